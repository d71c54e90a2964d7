"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel name, launches,
total and mean device time, and share of the listed time (our kernels only unless --all)."""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
skip_prefix = int(sys.argv[2]) if len(sys.argv) > 2 else 0      # ignore the first N launches (warm-up)
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    rows.append((int(r["ID"]), r["Kernel Name"], float(r["Metric Value"]), r.get("Metric Unit", "")))
rows = [x for x in rows if x[0] >= skip_prefix]
ours = [x for x in rows if any(k in x[1] for k in ("split", "combine", "kv_append", "rope", "rmsnorm", "silu"))]
tot = defaultdict(float)
cnt = defaultdict(int)
unit = rows[0][3] if rows else ""
for _, name, v, _ in ours:
    m = re.search(r"([A-Za-z_]\w*)(?:<[^()]*>)?\(", name)
    key = m.group(1) if m else name[:40]
    tot[key] += v
    cnt[key] += 1
T = sum(tot.values())
print(f"{path}: {len(ours)} of our launches ({unit})")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"  {k:40s} n={cnt[k]:4d} total={tot[k]:12.1f} mean={tot[k] / cnt[k]:10.2f} share={tot[k] / T:.3f}")
