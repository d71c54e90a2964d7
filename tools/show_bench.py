"""Summarise bench JSON lines: tok/s, ms/step, split us, roofline frac, split share, bounds, clocks."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as exc:
        print(p, "unreadable:", exc)
        continue
    r = d.get("roofline", {})
    b = r.get("bounds_us_per_launch", {})
    print(p.split("/")[-1], round(d["value"]), "tok/s", round(d["ms_per_step"], 3), "ms/step", "split_us",
          round(r.get("split_ms_per_launch", 0) * 1e3, 1), "frac", round(r.get("frac", 0), 3), "share",
          r.get("split_share_of_step") and round(r["split_share_of_step"], 3),
          {k: round(v, 1) for k, v in b.items() if k in ("hbm", "tensor_bf16", "mufu_ex2")},
          (d.get("clocks") or {}).get("sm_mhz"))
