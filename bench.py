#!/usr/bin/env python
"""bench.py — expansion tokens/s of Orion's content-parallel-expansion decode step on B200.

One "step" = one decode token for EVERY branch (key point) of every in-flight query, through
all L layers: per layer K1 kv_append, K2 split attention, K3 combine (
PAPER.md:337 Alg. 1 l.16).  Default workload = config c4 (BASELINE.json configs[3]: Llama-3-8B
attention shape, 64 queries x mixed16 DAG, 4K prefix, 512 tokens/point, 32 layers), the
8B-shaped config the north_star's >=70%-of-HBM target names.  Inputs are synthetic (seeded
N(0,1) bf16), every layer has its own KV pool, so each step's working set (~113 GB) is far
larger than L2 — no flush needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl orion|reference]

Multi-GPU: one process per GPU, no collective on the data path (queries are
independent).  `--gpus N` under torchrun (WORLD_SIZE=N) runs this process as
one rank; without WORLD_SIZE it launches the N ranks itself (torch.distributed.run, 127.0.0.1).
--scaling strong (default): the config's queries are partitioned over the ranks (c4: 64/N per
GPU, BASELINE configs[3] "queries partitioned across 2/4/8 B200"); --scaling weak: every rank
expands its own full batch.  Rank 0 prints one JSON line: the whole-job value (branches of all
ranks / max-over-ranks device-timed step) and every rank's own step time.  `--plan-only` runs
the launcher, sharding, planning and reductions without a GPU (gloo): the CPU test of this path.
`--impl reference` times the CPU oracle (the tier's reference arm) on a bounded sample.
"""
import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workloads import configs as WC, tensors as WT  # noqa: E402

METRIC = "expansion tokens/sec"
UNIT = "tokens/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(WC.CONFIGS))
    ap.add_argument("--impl", default="orion", choices=["orion", "reference"])
    ap.add_argument("--policy", type=int, default=0, help="0 ANCESTORS, 1 PARENTS_EQ3")
    ap.add_argument("--chunk", type=int, default=0, help="plan chunk_tokens (0 = default)")
    ap.add_argument("--kv-layout", default="separate", choices=["separate", "interleaved"],
                    help="KV cache layout: separate K / V pools, or K and V of a (page, kv head) adjacent")
    ap.add_argument("--no-merge", action="store_true",
                    help="plan without multi-range item merging (ORION_PLAN_NO_MERGE), for comparison")
    ap.add_argument("--unfused", action="store_true",
                    help="time the step as orion_kv_append + orion_expand_attn instead of orion_expand_step "
                         "(the append fused into the split launch), for A/B")
    ap.add_argument("--no-hybrid", action="store_true",
                    help="every decode item on the swap-AB kernel (ORION_PLAN_NO_HYBRID), for comparison")
    ap.add_argument("--kernel", default="tc", choices=["tc", "rol", "mma"],
                    help="split kernel: tcgen05 swap-AB (default), tcgen05 rows-on-lanes (rol) or legacy mma.sync")
    ap.add_argument("--layers", type=int, default=0, help="override layer count (0 = config)")
    ap.add_argument("--queries", type=int, default=0, help="override query count (0 = config)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default): the config's queries are split across ranks; weak: every "
                         "rank runs the full config")
    ap.add_argument("--plan-only", action="store_true",
                    help="launch, shard, plan and reduce without a GPU (gloo; CPU test of the N>1 path)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-model", action="store_true",
                    help="skip the whole-model step (random Llama-3-8B-shaped layers, SURVEY.md §8(f) rank 4)")
    ap.add_argument("--no-expansion", action="store_true",
                    help="skip the whole-expansion run (Alg. 1 l.9-22 driver, SURVEY.md §8(f) rank 2)")
    ap.add_argument("--no-point-prefill", action="store_true",
                    help="skip the point-prefill attention measurement (SURVEY.md §8(f) rank 1)")
    ap.add_argument("--no-prefill", action="store_true",
                    help="skip the co-scheduled prefill measurement (SURVEY.md §8(a) a8)")
    ap.add_argument("--no-shares", action="store_true",
                    help="skip the per-GPU shares of the strong-scaling curve (N=1 only)")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the c5 stress sub-results (wide-64 / chain-64, one GPU's 8-query share)")
    ap.add_argument("--prefill-caps", default="148,132,116",
                    help="split-kernel SM caps tried with the prefill co-stream")
    ap.add_argument("--green-splits", default="116,100,84",
                    help="expansion SM counts of the green-context partitions (prefill gets the rest)")
    return ap.parse_args(argv)


# ------------------------------------------------------------------------------ helpers
def algorithmic_bytes(cfg, lay):
    """Per layer: unique KV (each valid token row once per (query, kv head)),
    q read and out write.  Returns (kv_bytes, q_bytes, out_bytes)."""
    tokens = 0
    for qi in range(lay.n_queries):
        b0, n = int(lay.branch0[qi]), int(lay.n_points[qi])
        tokens += int(lay.prefix_len[qi]) + int(lay.own_len[b0:b0 + n].sum())
    kv = tokens * cfg.hkv * cfg.d * 2 * 2
    qb = lay.n_branches * cfg.hq * cfg.d * 2
    return kv, qb, qb


def context_tokens(batch):
    """Σ_b |ctx(b)| per kv head for the batch's current lengths (SURVEY.md §8(d) flops / exps)."""
    segs, own = batch.segs, batch.own_len.cpu().numpy()
    ln = segs["len"].astype(np.int64)
    dyn = segs["dyn"]
    m = dyn >= 0
    ln[m] = np.clip(own[dyn[m]] - segs["start"][m], 0, ln[m])
    return int(ln.sum())


def load_json(name):
    p = os.path.join(ROOT, name)
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def load_peaks():
    d = load_json("MEASURED_PEAKS.json")
    if "hbm_gbs" in d:
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config_name, kernel):
    """ncu DRAM bytes per split launch of this workload (profiles/ncu_traffic.json, from one
    `ncu --set full` capture), or None."""
    e = load_json(os.path.join("profiles", "ncu_traffic.json")).get(
        config_name if kernel == "tc" else f"{config_name}:{kernel}")
    return None if e is None else e.get("split_dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), "--query-gpu=" + self.FIELDS,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.3)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(", ") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[3:7]):
                if v.strip() == "Active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def host_cpu():
    """(usable cores, CPU model) of this host: the cores the process may run on
    (sched_getaffinity) and /proc/cpuinfo's model name."""
    cores = len(os.sched_getaffinity(0))
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return cores, model


# ------------------------------------------------------------------------------ oracle leg
def oracle_sample(cfg, seed):
    """One bounded sample of the workload on the CPU oracle: one query (all its points), one
    layer — K1 append (O4) of K and V, then the attention of every branch (O3).  Returns
    (seconds, branches)."""
    from oracle import append as OA, step as OS
    import torch
    lay = WT.make_layout(cfg, queries=[0], seed=seed, extra_tokens=0)
    ten = WT.make_qkv(cfg, lay, seed=seed)

    def u16(t):
        return t[0].contiguous().view(torch.int16).numpy().view(np.uint16)

    k, v, q, kn, vn = (u16(ten[x]) for x in ("k_cache", "v_cache", "q", "k_new", "v_new"))
    t0 = time.perf_counter()
    k2, own = OA.kv_append(k, kn, lay.page_table, lay.point_pt_off, lay.own_len, cfg.page, rewrite=True)
    v2, _ = OA.kv_append(v, vn, lay.page_table, lay.point_pt_off, lay.own_len, cfg.page, rewrite=True)
    OS.expand_step(lay, q, k2, v2, own_len=own)
    return time.perf_counter() - t0, lay.n_branches


def cpu_baseline(cfg, layers, seconds):
    """The oracle as it stands, on this host's cores (BLAS pinned to them with threadpoolctl), on a
    bounded sample: whole queries of the workload at one layer, extrapolated to `layers`."""
    from threadpoolctl import threadpool_limits
    cores, model = host_cpu()
    spent, n_br, n = 0.0, 0, 0
    with threadpool_limits(cores):
        while spent < seconds or n == 0:
            dt, br = oracle_sample(cfg, cfg.seed + 17 * n)
            spent += dt
            n_br += br
            n += 1
            if n >= 64:
                break
    # whole-job equivalent: each sampled (query, layer) would repeat for every layer
    value = n_br / (spent * layers)
    return {"value": value, "unit": UNIT, "cores": cores, "cpu_model": model, "kind": "oracle",
            "extrapolated": True, "blas_threads": cores,
            "sample": f"{n} x (1 query of {cfg.name}: append + attention of all its branches, "
                      f"1 layer), {spent:.1f} s CPU measured; rate extrapolated to {layers} layers"}


def workload_str(cfg, layers, world=1, scaling="strong"):
    """config.workload of both arms (the same workload; the reference arm times a sample of it)."""
    s = (f"{cfg.name}: Hq/Hkv/d={cfg.hq}/{cfg.hkv}/{cfg.d}, {cfg.n_queries} queries x {cfg.dag}, "
         f"prefix {cfg.lp}, {cfg.t} tok/point (Lc {cfg.lc}), page {cfg.page}, {layers} layers")
    if world > 1:
        s += (f"; queries partitioned over {world} GPUs" if scaling == "strong"
              else f"; each of {world} GPUs its own {cfg.n_queries}-query batch")
    return s


def run_reference(args, cfg, layers):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    cores, model = host_cpu()
    times, n_br = [], 0
    with threadpool_limits(cores):
        for s in range(args.warmup + args.steps):
            dt, br = oracle_sample(cfg, cfg.seed + 1000 + s)
            if s >= args.warmup:
                times.append(dt)
                n_br = br
    t_sample = statistics.mean(times)                  # measured seconds per step (1 query, 1 layer)
    value = n_br / (t_sample * layers)                 # extrapolated: every layer of one query
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_sample * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "extrapolated": True,
            "extrapolation": f"ms_per_step is the measured time of one step's sample (1 query x 1 layer: "
                             f"append + attention of its {n_br} branches); value = {n_br} branches / "
                             f"(that time x {layers} layers), the config's per-query rate (queries are "
                             f"independent)",
            "config": {"workload": workload_str(cfg, layers), "policy": "ancestors"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu_model": model,
                             "blas_threads": cores, "kind": "oracle", "extrapolated": True,
                             "sample": f"per step 1 query of {cfg.name} (all {n_br} branches), 1 layer, "
                                       f"append + attention, {t_sample:.2f} s measured; the rate scaled "
                                       f"by {layers} layers"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU leg
def plan_flags(args):
    import paper_2510_24390_b200 as orion
    return ({"tc": 0, "rol": orion.PLAN_ROWS_ON_LANES, "mma": orion.PLAN_MMA_SYNC}[args.kernel]
            | (orion.PLAN_NO_MERGE if args.no_merge else 0) | (orion.PLAN_NO_HYBRID if args.no_hybrid else 0))


def batch_of(args, cfg, lay, dev, **kw):
    import paper_2510_24390_b200 as orion
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    opts = dict(policy=args.policy, device=dev, chunk_tokens=args.chunk,
                kv_interleaved=args.kv_layout == "interleaved", flags=plan_flags(args))
    opts.update(kw)
    return orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                                lay.own_len, **opts)


def alloc_tensors(args, cfg, lay, layers, dev, seed):
    """Per-layer KV pools and per-step inputs, seeded N(0,1) bf16 on the device."""
    import torch
    B = lay.n_branches
    P, H, Hq, D = cfg.page, cfg.hkv, cfg.hq, cfg.d
    if args.kv_layout == "interleaved":          # one [pages][Hkv][2][P][d] pool per layer
        kv = torch.empty((layers, lay.num_pages, H, 2, P, D), dtype=torch.bfloat16, device=dev)
        kc, vc = kv[:, :, :, 0], kv[:, :, :, 1]
    else:
        kc = torch.empty((layers, lay.num_pages, H, P, D), dtype=torch.bfloat16, device=dev)
        vc = torch.empty_like(kc)
    q = torch.empty((layers, B, Hq, D), dtype=torch.bfloat16, device=dev)
    kn = torch.empty((layers, B, H, D), dtype=torch.bfloat16, device=dev)
    vn = torch.empty_like(kn)
    out = torch.empty_like(q)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    for t in (kc, vc, q, kn, vn):
        for l in range(layers):
            t[l].normal_(generator=g)
    return kc, vc, q, kn, vn, out


FUSED = True    # region A through orion_expand_step (--unfused: the three calls, for A/B)


def time_steps(batch, layers, tens, steps, warmup, stream, world=1, barrier=None):
    """Warm up, then two timed regions of `steps` steps each (per layer: append REWRITE, split,
    combine), CUDA events on `stream`:
      A (the headline): per layer one orion_expand_step (the append runs inside the split launch
        where the plan allows), events only at step boundaries -- an event recorded between two
        kernels breaks their programmatic-dependent-launch edge (≈ 2 % of the c4 step), so none is;
      B (the kernel timing): the same steps as three calls (append, split, combine) with events
        around every split launch, for the split kernel's average launch duration (the roofline)
        and its share of B's step time.
    Returns (elapsed_ms A, per-step ms A sorted, per-launch split ms B, elapsed_ms B, launches, step)."""
    import torch
    import paper_2510_24390_b200 as orion
    kc, vc, q, kn, vn, out = tens
    REW = orion.APPEND_REWRITE

    def step(ev=None, k=0):
        if ev is None and FUSED:   # the public call: orion_expand_step (append in the split launch)
            for l in range(layers):
                batch.step(q[l], kn[l], vn[l], kc[l], vc[l], out[l], mode=REW)
            return
        if ev is None:
            for l in range(layers):
                batch.append(kn[l], vn[l], kc[l], vc[l], mode=REW)
                batch.split(q[l], kc[l], vc[l])
                batch.combine(out[l])
            return
        for l in range(layers):
            batch.append(kn[l], vn[l], kc[l], vc[l], mode=REW)
            ev[k][l][0].record(stream)
            batch.split(q[l], kc[l], vc[l])
            ev[k][l][1].record(stream)
            batch.combine(out[l])

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    # ---- region A
    if barrier:
        barrier()
    torch.cuda.synchronize()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    step_ev[0].record(stream)
    for k in range(steps):
        step()
        step_ev[k + 1].record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    elapsed_a = step_ev[0].elapsed_time(step_ev[steps])
    step_ms = sorted(step_ev[k].elapsed_time(step_ev[k + 1]) for k in range(steps))
    # ---- region B
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(layers)] for _ in range(steps)]
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0.record(stream)
    for k in range(steps):
        step(ev, k)
    b1.record(stream)
    torch.cuda.synchronize()
    split_ms = [ev[k][l][0].elapsed_time(ev[k][l][1]) for k in range(steps) for l in range(layers)]
    nb = batch.stats.get("n_big", 0)
    # region A's launches per layer: orion_step_launches (2 when orion_expand_step fuses the
    # append into the split launch, else append + split kernel(s) + combine)
    n_kernels = batch.step_launches() if FUSED else 3 + (1 if 0 < nb < batch.stats["n_items"] else 0)
    return elapsed_a, step_ms, split_ms, b0.elapsed_time(b1), steps * layers * n_kernels, step


def bounds_of(cfg, lay, batch, split_bytes):
    """three bounds per split launch -- bytes / HBM, flops / tensor, exps / MUFU."""
    peaks_all = load_json("MEASURED_PEAKS.json")
    sm_mhz = peaks_all.get("sm_max_mhz", 1965.0)
    ctx_tok = context_tokens(batch)
    flops = 4.0 * cfg.d * cfg.hq * ctx_tok
    exps = float(cfg.hq * ctx_tok)
    return {"hbm": split_bytes / (load_peaks()[0] * 1e9) * 1e6,
            "tensor_bf16": flops / (peaks_all.get("bf16_tflops", 2250.0) * 1e12) * 1e6,
            "mufu_ex2": exps / (16 * 148 * sm_mhz * 1e6) * 1e6,
            "flops": flops, "exps": exps,
            "note": "MUFU: 16 ex2/clk/SM x 148 SMs at the max SM clock"}


def plan_only(args, cfg, layers):
    """The N>1 host path without a GPU: rank launch, query sharding, per-rank layouts and plans,
    the max/sum reductions and the per-rank gather over torch.distributed (gloo), and rank 0's
    JSON line.  Nothing is timed (value null)."""
    import torch.distributed as dist
    import paper_2510_24390_b200 as orion
    from paper_2510_24390_b200 import shard
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    qs = shard.rank_queries(cfg.n_queries, rank, world, args.scaling)
    lay = WT.make_layout(cfg, queries=qs, seed=shard.rank_seed(cfg.seed, rank))
    t0 = time.perf_counter()
    batch = batch_of(args, cfg, lay, "cpu")
    plan_s = time.perf_counter() - t0
    kv_b, q_b, _ = algorithmic_bytes(cfg, lay)
    mine = {"rank": rank, "queries": qs, "branches": lay.n_branches, "plan_s": plan_s,
            "items": batch.stats["n_items"], "kv_bytes_per_layer": kv_b}
    plan_s_max, total_b = shard.reduce_timing(plan_s, float(lay.n_branches))
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": 0,
                          "warmup": 0, "ms_per_step": None, "higher_is_better": True,
                          "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
                          "data": "synthetic", "plan_only": True,
                          "config": {"workload": workload_str(cfg, layers, world, args.scaling),
                                     "branches_per_step": int(total_b), "layers": layers},
                          "plan_s_max": plan_s_max, "per_rank": per_rank,
                          "gpu_launches": 0}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_orion(args, cfg, layers):
    import torch
    import torch.distributed as dist
    import paper_2510_24390_b200 as orion
    from paper_2510_24390_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    barrier = dist.barrier if world > 1 else None

    qs = shard.rank_queries(cfg.n_queries, rank, world, args.scaling)
    lay = WT.make_layout(cfg, queries=qs, seed=shard.rank_seed(cfg.seed, rank))
    B = lay.n_branches
    tens = alloc_tensors(args, cfg, lay, layers, dev, cfg.seed * 7 + rank)
    kc, vc, q, kn, vn, out = tens
    t0 = time.perf_counter()
    batch = batch_of(args, cfg, lay, dev)
    plan_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream(dev)
    sampler = ClockSampler(local) if rank == 0 else None
    elapsed_ms, step_ms, split_ms, elapsed_b, launches, step = time_steps(batch, layers, tens, args.steps,
                                                                          args.warmup, stream, world, barrier)
    clocks = sampler.stop() if sampler else None
    pct = lambda f: step_ms[min(len(step_ms) - 1, int(round(f * (len(step_ms) - 1))))]
    my_ms = elapsed_ms
    # whole-job aggregation: branches of all ranks / max step time over ranks
    elapsed_ms, total_b = shard.reduce_timing(elapsed_ms, float(B), device=dev)
    ms_step = elapsed_ms / args.steps
    value = total_b / (ms_step / 1e3)
    per_rank = [{"rank": rank, "queries": len(qs), "branches": B, "ms_per_step": my_ms / args.steps}]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, {"rank": rank, "queries": len(qs), "branches": B,
                                          "ms_per_step": my_ms / args.steps})

    # ---- the same step captured once as a CUDA graph and replayed (SURVEY.md §8(d) protocol)
    graph = None
    try:
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            step()                                     # warm the capture stream
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, stream=gs):
            step()
        for _ in range(max(3, args.warmup)):
            cg.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            cg.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gms, _ = shard.reduce_timing(g0.elapsed_time(g1), 0.0, device=dev)
        graph = {"ms_per_step": gms / args.steps, "tokens_per_s": total_b / (gms / args.steps / 1e3),
                 "note": f"one step ({layers} layers x orion_expand_step) captured once, replayed {args.steps}x"}
        del cg
    except Exception as exc:                             # capture unsupported here: say so
        graph = {"unavailable": f"{type(exc).__name__}: {exc}"}

    # ---- end to end through the public API with host buffers (pinned), copies inside timing
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, batch, layers, q, kn, vn, out, kc, vc, dev, world, total_b)

    kv_b, q_b, o_b = algorithmic_bytes(cfg, lay)
    split_bytes = kv_b + q_b                        # K2 reads: unique KV + q
    split_avg_s = statistics.mean(split_ms) / 1e3
    peak, peak_src = load_peaks()
    achieved = split_bytes / split_avg_s / 1e9
    st = batch.stats
    costream = None
    if world > 1 and not args.no_prefill:           # c4 "with co-scheduled prefill stream": every rank
        mine = run_costream(args, cfg, lay, layers, q, kn, vn, out, kc, vc, dev, B / (my_ms / args.steps / 1e3))
        allc = [None] * world
        dist.all_gather_object(allc, mine)
        costream = {"per_rank": allc,
                    "expansion_tok_s_together_cap148_total": sum(
                        c["together"][0]["expansion_tok_s"] for c in allc if c and c.get("together")),
                    "note": "each rank runs the co-stream experiment on its own GPU and query share"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) bf16 q/K/V; random page permutation)",
        "config": {"workload": workload_str(cfg, layers, world, args.scaling),
                   "branches_per_step": int(total_b), "layers": layers,
                   "policy": "parents_eq3" if args.policy else "ancestors",
                   "append_mode": "rewrite (stationary snapshot)",
                   "kv_layout": args.kv_layout,
                   "l2": "no flush: per-layer KV pools, step working set "
                         f"{layers * (kv_b + q_b + o_b) / 1e9:.1f} GB per GPU >> 126 MB L2",
                   "parallelism": (f"{cfg.n_queries} queries partitioned over {world} GPU(s) "
                                   f"({cfg.n_queries // world if world <= cfg.n_queries else 0}+ per GPU), no collective"
                                   if args.scaling == "strong" else
                                   f"{world} GPU(s), each its own {cfg.n_queries}-query batch, no collective")},
        "roofline": {"bound": "hbm",
                     "kernel": {"tc": "split_tct_kernel (K2, tcgen05 swap-AB) + split_tc_kernel on hybrid big items",
                                "rol": "split_tc_kernel (K2, tcgen05 rows-on-lanes)",
                                "mma": "split_kernel (K2, mma.sync)"}[args.kernel],
                     "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": load_traffic(cfg.name, args.kernel),
                     "frac_of_nominal_8tbs": achieved / 8000.0,
                     "bounds_us_per_launch": bounds_of(cfg, lay, batch, split_bytes),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": split_bytes,
                     "split_ms_per_launch": split_avg_s * 1e3,
                     "split_share_of_step": sum(split_ms) / elapsed_b,
                     # the same split launches against the headline step (region A, no inner events):
                     # what the rest of a layer (append, combine, launch edges) costs the headline
                     "split_share_of_headline_step": split_avg_s * 1e3 * layers / ms_step,
                     "timing_note": "value / ms_per_step: timed region A, events only at step boundaries; "
                                    "split_ms_per_launch: region B, the same steps with events around every "
                                    "split launch (those events cost ~2 % of the step: they break the "
                                    "programmatic-dependent-launch edges)",
                     "region_b_ms_per_step": elapsed_b / args.steps,
                     "rank": 0,
                     "step_gbs_all_kernels": layers * (kv_b + q_b + o_b) / (ms_step / 1e3) / 1e9},
        "plan": {"items": st["n_items"], "big_items": st.get("n_big", 0), "pieces": st["n_pieces"],
                 "partials": st["n_partials"],
                 "unique_tokens_per_kvhead": st["unique_tokens"],
                 "logical_tokens_per_kvhead": st["logical_tokens"],
                 "partial_bytes_per_layer": st["workspace_bytes"] * 2,   # written by K2 + read by K3
                 "plan_build_s": plan_s},
        "per_rank": per_rank,
        "step_ms": {"p10": pct(0.1), "median": pct(0.5), "p90": pct(0.9), "rank0_only": world > 1},
        "cuda_graph": graph,
        "per_layer": {"us": ms_step / layers * 1e3, "tokens_per_s": float(total_b) / (ms_step / layers / 1e3)},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
    }
    if costream is not None:
        line["prefill_costream"] = costream
    if world == 1:
        line["contiguous_pages"] = run_contiguous(args, cfg, lay, layers, q, kc, vc, out, dev)
    if world == 1 and not args.no_shares and args.scaling == "strong" and cfg.n_queries >= 16:
        line["strong_scaling_shares"] = run_shares(args, cfg, lay, layers, tens, dev, value)
    if world == 1 and not args.no_model:
        line["model_step"] = run_model_step(args, cfg, lay, layers, kc, vc, dev, value)
    if world == 1 and not args.no_expansion:
        line["expansion_run"] = run_expansion(args, cfg, lay, layers, q, kn, vn, kc, vc, dev)
        if cfg.name == "c4":
            line["expansion_run_c2"] = run_expansion_small(args, dev)
    if world == 1 and not args.no_point_prefill:
        line["point_prefill"] = run_point_prefill(args, cfg, lay, layers, kc, vc, dev)
    if world == 1 and not args.no_prefill:
        line["prefill_costream"] = run_costream(args, cfg, lay, layers, q, kn, vn, out, kc, vc, dev,
                                                value)
    if world == 1 and not args.no_c5 and cfg.name == "c4":
        del batch, tens, kc, vc, q, kn, vn, out
        torch.cuda.empty_cache()
        line["c5"] = run_c5(args, dev)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, layers, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_shares(args, cfg, lay, layers, tens, dev, full_value):
    """The single-GPU points of the strong-scaling curve: the step on the first Q/N queries of the
    batch (what one rank of an N-GPU run expands, same pools), N = 2, 4, 8.  projected_value =
    N x its rate (ranks share nothing)."""
    import torch
    kc, vc, q, kn, vn, out = tens
    res = {}
    for n in (2, 4, 8):
        nq = cfg.n_queries // n
        if nq < 1:
            continue
        sub, br = WT.subset_layout(lay, list(range(nq)))
        idx = torch.from_numpy(br).to(dev)
        sub_t = (kc, vc, q.index_select(1, idx), kn.index_select(1, idx), vn.index_select(1, idx),
                 out.index_select(1, idx))
        batch = batch_of(args, cfg, sub, dev)
        steps = max(3, min(args.steps, 10))
        ms, _, split_ms, _, _, _ = time_steps(batch, layers, sub_t, steps, 2, torch.cuda.current_stream(dev))
        tok_s = sub.n_branches / (ms / steps / 1e3)
        res[f"n{n}"] = {"queries_per_gpu": nq, "branches_per_gpu": sub.n_branches,
                        "ms_per_step": ms / steps, "tokens_per_s_per_gpu": tok_s,
                        "split_ms_per_launch": statistics.mean(split_ms),
                        "projected_value": n * tok_s, "projected_efficiency": n * tok_s / (n * full_value)}
    return res


def run_c5(args, dev):
    """BASELINE configs[4] (the stress config): one GPU's share of the 8-GPU run, 8 queries x wide-64
    and 8 queries x chain-64 (8K prefix, 256 tok/point, 32 layers), the default plan; tok/s, the
    split kernels' time against the three bounds and ncu's DRAM bytes."""
    import torch
    res = {}
    for name in ("c5w", "c5c"):
        cfg = WC.CONFIGS[name].with_(n_queries=8)
        layers = cfg.layers
        lay = WT.make_layout(cfg, seed=cfg.seed)
        tens = alloc_tensors(args, cfg, lay, layers, dev, cfg.seed * 7)
        batch = batch_of(args, cfg, lay, dev)
        steps = max(3, min(args.steps, 10))
        ms, _, split_ms, _, _, _ = time_steps(batch, layers, tens, steps, 3, torch.cuda.current_stream(dev))
        kv_b, q_b, _ = algorithmic_bytes(cfg, lay)
        split_s = statistics.mean(split_ms) / 1e3
        b = bounds_of(cfg, lay, batch, kv_b + q_b)
        peak, _ = load_peaks()
        bound_us = max(b["hbm"], b["tensor_bf16"], b["mufu_ex2"])
        res[f"{name}_8q"] = {
            "workload": workload_str(cfg, layers) + " (one GPU's share of 64 queries on 8 GPUs)",
            "tokens_per_s": lay.n_branches / (ms / steps / 1e3), "ms_per_step": ms / steps,
            "split_us_per_launch": split_s * 1e6, "split_gbs": (kv_b + q_b) / split_s / 1e9,
            "frac_of_hbm_peak": (kv_b + q_b) / split_s / 1e9 / peak,
            "bounds_us": {k: b[k] for k in ("hbm", "tensor_bf16", "mufu_ex2")},
            "frac_of_max_bound": bound_us / (split_s * 1e6),
            "ncu_dram_bytes_per_launch": load_traffic(name, args.kernel),
            "plan": {"items": batch.stats["n_items"], "big_items": batch.stats.get("n_big", 0),
                     "partials": batch.stats["n_partials"]}}
        del tens, batch
        torch.cuda.empty_cache()
    return res


def run_contiguous(args, cfg, lay, layers, q, kc, vc, out, dev):
    """SURVEY.md §8(d) variant: the same step with every page run physically contiguous (page
    table = identity over the same pools) instead of a random page permutation."""
    import torch
    import paper_2510_24390_b200 as orion
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    ident = np.arange(len(lay.page_table), dtype=np.int32)
    batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, ident,
                                 lay.own_len, policy=args.policy, device=dev, chunk_tokens=args.chunk, kv_interleaved=args.kv_layout == "interleaved")
    stream = torch.cuda.current_stream(dev)
    for l in range(min(3, layers)):
        batch.attend(q[l], out[l], kc[l], vc[l])
    torch.cuda.synchronize()
    n = max(3, min(args.steps, 10))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n * layers)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(n):
        for l in range(layers):
            evs[i * layers + l][0].record(stream)
            batch.split(q[l], kc[l], vc[l])
            evs[i * layers + l][1].record(stream)
            batch.combine(out[l])
    e1.record(stream)
    torch.cuda.synchronize()
    split_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    kv_b, q_b, _ = algorithmic_bytes(cfg, lay)
    ms = e0.elapsed_time(e1) / n
    return {"note": "attention only (split + combine per layer, no append), contiguous page runs",
            "tokens_per_s": lay.n_branches / (ms / 1e3), "ms_per_step": ms,
            "split_ms_per_launch": split_ms, "split_gbs": (kv_b + q_b) / (split_ms / 1e3) / 1e9}


def run_model_step(args, cfg, lay, layers, kc, vc, dev, attention_only):
    """§8(f) rank 4: the whole-model expansion step -- every branch generates one token through
    `layers` Llama-3-8B-shaped decoder layers with random weights (hidden 4096, 32 / 8 heads of 128,
    SwiGLU 14336): per layer RMSNorm, QKV GEMM, RoPE fused into the KV append, the expansion
    attention, O GEMM, RMSNorm, gate|up GEMM, SiLU*up, down GEMM (GEMMs: cuBLAS; the rest: orion
    kernels).  The paper's metric is exactly this: generated tokens / s.  The KV
    slot is rewritten (REWRITE) so the snapshot stays stationary across steps."""
    import torch
    import paper_2510_24390_b200 as orion
    from paper_2510_24390_b200.model import DecoderModel
    hidden, inter = 4096, 14336
    model = DecoderModel(layers, hidden, cfg.hq, cfg.hkv, cfg.d, inter, device=dev, seed=11, init_scale=0.5)
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                                 lay.own_len, policy=args.policy, device=dev, chunk_tokens=args.chunk,
                                 kv_interleaved=args.kv_layout == "interleaved")
    B = lay.n_branches
    pos_base = torch.from_numpy(batch.pos_base()).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed * 19)
    x = torch.randn((B, hidden), generator=g, device=dev).to(torch.bfloat16)
    buf = model.buffers(B, dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(2):
        y = model.step(x, batch, kc[:layers], vc[:layers], pos_base, buf, first_mode=orion.APPEND_REWRITE)
    torch.cuda.synchronize()
    n = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        y = model.step(x, batch, kc[:layers], vc[:layers], pos_base, buf, first_mode=orion.APPEND_REWRITE)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    finite = bool(torch.isfinite(y.float()).all().item())
    gemm_flop = model.flops_per_token() * B
    return {"workload": f"{cfg.name}: {B} branches x {layers} decoder layers (hidden {hidden}, "
                        f"{cfg.hq}/{cfg.hkv} heads of {cfg.d}, SwiGLU {inter}), random weights",
            "metric": "generated tokens/sec (whole model)", "value": B / (ms / 1e3), "unit": "tokens/s",
            "ms_per_step": ms, "steps": n, "weights_gb": model.weight_bytes() / 1e9,
            "gemm_tflop_per_step": gemm_flop / 1e12,
            "attention_only_tok_s": attention_only,
            "attention_share_est": (B / attention_only) / (ms / 1e3) if attention_only else None,
            "output_finite": finite}


def expansion_decode_bytes(cfg, lay, ex, schedule, layers):
    """Algorithmic HBM bytes of the decode rounds of a whole expansion (SURVEY.md 8(d)'s formula per
    round).  Replays the lengths: a round's attention sees each running branch's own segment with
    the token just appended.  A point's spans (CONTENT [0, Lc), FULL [0, T), OUTPUT [Lc, T), OWN
    [0, own)) and the prefix [0, Lp) overlap or touch, so a page run's union is max end - min start."""
    so, sg = ex.seg_offsets, ex.segs
    own = np.full(ex.n_branches, cfg.lc, np.int64)
    per_tok = cfg.hkv * cfg.d * 2 * 2
    total = 0
    for dec in schedule:
        cur = own.copy()
        cur[dec] += 1
        idx = np.concatenate([np.arange(so[b], so[b + 1]) for b in dec])
        seg = sg[idx]
        dyn = seg["dyn"].astype(np.int64)
        ln = seg["len"].astype(np.int64)
        eff = np.where(dyn >= 0, np.clip(cur[np.maximum(dyn, 0)] - seg["start"], 0, ln), ln)
        keep = eff > 0
        pt, st, en = seg["pt_off"][keep], seg["start"][keep].astype(np.int64), (seg["start"][keep] + eff[keep])
        order = np.argsort(pt, kind="stable")
        pt, st, en = pt[order], st[order], en[order]
        starts = np.flatnonzero(np.r_[True, pt[1:] != pt[:-1]])
        uniq = int((np.maximum.reduceat(en, starts) - np.minimum.reduceat(st, starts)).sum())
        total += layers * (uniq * per_tok + len(dec) * cfg.hq * cfg.d * 2 * 2)
        own[dec] += 1
    return total


def run_expansion(args, cfg, lay, layers, q, kn, vn, kc, vc, dev, graph=True):
    """§8(f) rank 2: a whole expansion of the config's queries (Alg. 1 l.9-22 with
    continuous batching, reading D1): rounds of orion_expansion_round; each round prefills the
    points that became ready (orion_point_prefill_attn, every layer) and decodes one token of the
    running set through all layers (append + split + combine); plans are rebuilt only when the
    running set changes.  Every point generates T - Lc tokens.  graph=True replays each decode
    round from a CUDA graph captured once per running set (Expansion.decode).  Device-timed end
    to end (host scheduling, plan rebuilds, graph captures and the per-set input gathers inside
    the timed region)."""
    import torch
    from paper_2510_24390_b200.expansion import Expansion
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    B, lc = lay.n_branches, cfg.lc
    tokens = (np.asarray(lay.own_len) - lc).astype(np.int32)          # T - Lc per point
    ex = Expansion(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table, lc, tokens,
                   policy=args.policy, device=dev, chunk_tokens=args.chunk,
                   kv_interleaved=args.kv_layout == "interleaved")
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed * 17)
    q_pre = torch.randn((B, lc, cfg.hq, cfg.d), generator=g, device=dev).to(torch.bfloat16)
    out_pre = torch.empty_like(q_pre)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    rounds, dec_sum, pre_rounds, cur, subs = 0, 0, 0, None, None
    schedule = []                                  # running set of every decode round
    while True:
        pre, dec = ex.next_round()
        if len(pre) == 0 and len(dec) == 0:
            break
        if len(pre):
            idx = torch.from_numpy(pre.astype(np.int64)).to(dev)
            qp = q_pre.index_select(0, idx)
            op = out_pre[:len(pre)]
            ex.prefill(pre, [qp] * layers, kc[:layers], vc[:layers], [op] * layers)
            pre_rounds += 1
        if len(dec):
            if cur is None or len(cur) != len(dec) or not np.array_equal(cur, dec):
                idx = torch.from_numpy(dec.astype(np.int64)).to(dev)
                subs = [t.index_select(1, idx) for t in (q, kn, vn)]
                subs.append(torch.empty_like(subs[0]))
                cur = dec.copy()
            ex.decode(dec, subs[0], subs[1], subs[2], kc[:layers], vc[:layers], subs[3], graph=graph)
            dec_sum += len(dec)
            schedule.append(dec)
        rounds += 1
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    gen = int(tokens.sum())
    kv_bytes = expansion_decode_bytes(cfg, lay, ex, schedule, layers)
    peak, peak_src = load_peaks()
    return {"workload": f"{cfg.name}: whole expansion of {lay.n_queries} queries x {cfg.dag}, "
                        f"every point prefills Lc {lc} tokens then decodes T - Lc = {int(tokens.max())} "
                        f"tokens through {layers} layers",
            "metric": "expansion tokens/sec (whole expansion)", "value": gen / (ms / 1e3), "unit": "tokens/s",
            "generated_tokens": gen, "rounds": rounds, "rounds_with_prefill": pre_rounds,
            "mean_running_set": dec_sum / max(1, rounds), "max_branches": B,
            "plan_rebuilds": ex.rebuilds, "decode_graph": graph, "graph_captures": ex.captures,
            "ms": ms, "wall_ms": wall * 1e3, "us_per_round": ms * 1e3 / max(1, rounds),
            "roofline": {"bound": "hbm", "algorithmic_bytes": kv_bytes, "achieved": kv_bytes / (ms / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s", "frac": kv_bytes / (ms / 1e3) / 1e9 / peak,
                         "peak_source": peak_src,
                         "note": "all decode rounds: per round and layer, every (query, kv head)'s unique "
                                 "context tokens (union of its running branches' spans at their current "
                                 "lengths) x d x 2 (K, V) x 2 B, plus q read and out write (SURVEY.md "
                                 "8(d)); prefill rounds, appends and plan rebuilds count as time only"},
            "note": "device-timed (events) around the whole loop; host scheduling and plan "
                    "rebuilds inside; compare the snapshot value where every point decodes at once"}


def run_expansion_small(args, dev):
    """The latency-bound end of §8(f) rank 2: a whole expansion of BASELINE configs[1] (c2: one
    query, 8 points, 2K prefix, 256 tok/point, 32 layers), each decode round launched eagerly
    (3 launches per layer from the host) and replayed from a per-running-set CUDA graph."""
    import torch
    cfg = WC.CONFIGS["c2"]
    lay = WT.make_layout(cfg, seed=cfg.seed)
    kc, vc, q, kn, vn, _ = alloc_tensors(args, cfg, lay, cfg.layers, dev, cfg.seed * 7)
    res = {}
    for graph in (False, True):
        run_expansion(args, cfg, lay, cfg.layers, q, kn, vn, kc, vc, dev, graph=graph)   # warm-up
        r = run_expansion(args, cfg, lay, cfg.layers, q, kn, vn, kc, vc, dev, graph=graph)
        res["graph" if graph else "eager"] = r
    res["graph_speedup"] = res["graph"]["value"] / res["eager"]["value"]
    del kc, vc, q, kn, vn
    torch.cuda.empty_cache()
    return res


def run_point_prefill(args, cfg, lay, layers, kc, vc, dev):
    """§8(f) rank 1: the Pre-stage attention of every point of the batch (Alg. 1 l.12/19):
    Lc content rows per point attend to the point's dependency context plus their own content,
    causally (orion_point_prefill_attn; oracle O5).  Dense multi-row attention: tensor-bound.
    Timed on the device over `steps` launches cycling through the layers' KV pools."""
    import torch
    import paper_2510_24390_b200 as orion
    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    lc = cfg.lc
    batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                                 lay.own_len, policy=args.policy, device=dev, prefill_rows=lc, kv_interleaved=args.kv_layout == "interleaved")
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed * 13)
    B = lay.n_branches
    q = torch.randn((B, lc, cfg.hq, cfg.d), generator=g, device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    stream = torch.cuda.current_stream(dev)
    for l in range(min(3, layers)):
        batch.attend(q, out, kc[l], vc[l])
    torch.cuda.synchronize()
    n = max(3, min(args.steps, layers))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(n):
        batch.attend(q, out, kc[i % layers], vc[i % layers])
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    st = batch.stats
    # useful FLOPs (causal, no padding): per (branch, content row i, q head): (ctx_b + i + 1)
    # key rows x d x 4 (QK^T and PV).  logical_tokens = sum_b (ctx_b + Lc) per kv head.
    ctx_sum = st["logical_tokens"] - B * lc
    flop = cfg.hq * cfg.d * 4.0 * (lc * ctx_sum + B * lc * (lc + 1) / 2)
    tflops = flop / (ms / 1e3) / 1e12
    peaks = {}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            peaks = json.load(f)
    peak = peaks.get("bf16_tflops", 2250.0)
    return {"workload": f"{cfg.name} point prefill: {B} points x Lc {lc} content rows x {cfg.hq} heads, "
                        f"contexts = dependency lists + causal own ({args.policy and 'parents_eq3' or 'ancestors'})",
            "kernel": "split_tc_kernel (rows-on-lanes tcgen05, causal own items) + combine",
            "ms_per_layer": ms, "launches": n, "rows": B * lc * cfg.hq,
            "roofline": {"bound": "tensor", "achieved": tflops, "peak": peak, "unit": "TFLOP/s",
                         "frac": tflops / peak, "flop_per_launch": flop,
                         "peak_source": "measured (MEASURED_PEAKS.json bf16_tflops, burst)"
                                        if "bf16_tflops" in peaks else "nominal dense bf16"},
            "plan": {"items": st["n_items"], "partials": st["n_partials"]}}


# Llama-3-8B decoder-layer prefill of 4096 tokens: QKV, O, gate+up, down.
PREFILL_TOKENS = 4096
PREFILL_GEMMS = ((4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096))   # (K, N) of x[T,K]·W[K,N]


def run_costream(args, cfg, lay, layers, q, kn, vn, out, kc, vc, dev, expansion_alone):
    """§8(a) a8: KPG prefill of other queries as a compute-bound load on a low-priority stream
    (plain library GEMMs: torch.matmul -> cuBLAS/cuBLASLt, bf16) while the expansion step runs on
    a high-priority stream (decode is memory-bound, prefill compute-bound).
    Three cases: expansion alone (the headline run), prefill alone, both together -- the latter
    also with the persistent split kernel capped to fewer SMs (plan opts num_sms), leaving the
    rest to the GEMMs.  Device-timed with events on each stream."""
    import torch
    import paper_2510_24390_b200 as orion
    hi = torch.cuda.Stream(dev, priority=-1)
    lo = torch.cuda.Stream(dev, priority=0)
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    acts = {k: torch.randn((PREFILL_TOKENS, k), generator=g, device=dev, dtype=torch.bfloat16)
            for k in {k for k, _ in PREFILL_GEMMS}}
    ws = [torch.randn((k, n), generator=g, device=dev, dtype=torch.bfloat16) * 0.02
          for k, n in PREFILL_GEMMS]
    outs = [torch.empty((PREFILL_TOKENS, n), device=dev, dtype=torch.bfloat16) for _, n in PREFILL_GEMMS]
    gemm_flop = sum(2.0 * PREFILL_TOKENS * k * n for k, n in PREFILL_GEMMS)
    # ... plus the Pre-stage attention (§8(f) rank 1, orion_point_prefill_attn) of enough points
    # that their content rows match the GEMMs' token count: the first queries' points, each Lc
    # rows attending to its dependency context plus its own content (reads this layer pool)
    lc = cfg.lc
    n_pq = 0
    rows = 0
    while n_pq < lay.n_queries and rows < PREFILL_TOKENS:
        rows += int(lay.n_points[n_pq]) * lc
        n_pq += 1
    psub, _ = WT.subset_layout(lay, list(range(n_pq)))
    pqueries = [dict(n_points=int(psub.n_points[i]), edges=psub.edges[i],
                     prefix_pt_off=int(psub.prefix_pt_off[i]), prefix_len=int(psub.prefix_len[i]))
                for i in range(psub.n_queries)]
    ppoints = np.stack([psub.point_pt_off, psub.content_len, psub.point_cap], 1)

    def prefill_batch(cap):
        return orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, pqueries, ppoints, psub.page_table,
                                    psub.own_len, policy=args.policy, device=dev, num_sms=cap,
                                    prefill_rows=lc, kv_interleaved=args.kv_layout == "interleaved")

    pbatch = prefill_batch(0)
    qpf = torch.randn((psub.n_branches, lc, cfg.hq, cfg.d), generator=g, device=dev).to(torch.bfloat16)
    opf = torch.empty_like(qpf)
    pst = pbatch.stats
    ctx_sum = pst["logical_tokens"] - psub.n_branches * lc
    attn_flop = cfg.hq * cfg.d * 4.0 * (lc * ctx_sum + psub.n_branches * lc * (lc + 1) / 2)
    layer_flop = gemm_flop + attn_flop
    pf_pool = layers - 1                               # decode rewrites own slots only: benign reads

    def prefill_layer(pb=None):
        for (k, _), w, o in zip(PREFILL_GEMMS, ws, outs):
            torch.matmul(acts[k], w, out=o)
        (pb or pbatch).attend(qpf, opf, kc[pf_pool], vc[pf_pool])

    # prefill alone
    with torch.cuda.stream(lo):
        for _ in range(5):
            prefill_layer()
    torch.cuda.synchronize()
    n_alone = 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(lo)
    with torch.cuda.stream(lo):
        for _ in range(n_alone):
            prefill_layer()
    e1.record(lo)
    torch.cuda.synchronize()
    prefill_ms = e0.elapsed_time(e1) / n_alone
    prefill_alone = layer_flop / (prefill_ms / 1e3) / 1e12

    queries = [dict(n_points=int(lay.n_points[i]), edges=lay.edges[i],
                    prefix_pt_off=int(lay.prefix_pt_off[i]), prefix_len=int(lay.prefix_len[i]))
               for i in range(lay.n_queries)]
    points = np.stack([lay.point_pt_off, lay.content_len, lay.point_cap], 1)
    steps = max(3, min(args.steps, 10))
    REW = orion.APPEND_REWRITE
    together = []
    for cap in [int(c) for c in args.prefill_caps.split(",") if c]:
        batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points, lay.page_table,
                                     lay.own_len, policy=args.policy, device=dev,
                                     chunk_tokens=args.chunk, num_sms=cap, kv_interleaved=args.kv_layout == "interleaved")

        def step():
            for l in range(layers):
                batch.step(q[l], kn[l], vn[l], kc[l], vc[l], out[l], mode=REW, stream=hi)

        with torch.cuda.stream(hi):
            step()
        torch.cuda.synchronize()
        # expansion alone at this cap
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(hi)
        for _ in range(steps):
            step()
        a1.record(hi)
        torch.cuda.synchronize()
        exp_cap_ms = a0.elapsed_time(a1) / steps
        # together: enough prefill layers queued on `lo` to outlast the expansion window
        n_pf = int(steps * exp_cap_ms / prefill_ms * 1.5) + 4
        s_hi = torch.cuda.Event(enable_timing=True)
        s_lo = torch.cuda.Event(enable_timing=True)
        t_hi = torch.cuda.Event(enable_timing=True)
        pf_ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_pf)]
        torch.cuda.synchronize()
        s_lo.record(lo)
        with torch.cuda.stream(lo):
            for i in range(n_pf):
                prefill_layer()
                pf_ev[i].record(lo)
        s_hi.record(hi)
        for _ in range(steps):
            step()
        t_hi.record(hi)
        torch.cuda.synchronize()
        win = s_hi.elapsed_time(t_hi)
        lag = s_lo.elapsed_time(s_hi)                 # lo started this much earlier
        done = sum(1 for ev in pf_ev if lag <= s_lo.elapsed_time(ev) <= lag + win)
        exp_tok_s = lay.n_branches * steps / (win / 1e3)
        pf_tflops = done * layer_flop / (win / 1e3) / 1e12
        together.append({"split_sm_cap": cap, "expansion_alone_tok_s": lay.n_branches / (exp_cap_ms / 1e3),
                         "expansion_tok_s": exp_tok_s, "expansion_retained": exp_tok_s / expansion_alone,
                         "prefill_tflops": pf_tflops, "prefill_retained": pf_tflops / prefill_alone,
                         "prefill_layers_in_window": done})
    # §8(f) rank 3: the same two workloads on disjoint SM partitions (green contexts).
    partitioned = []
    try:
        from paper_2510_24390_b200.partition import SmPartition
        for n_exp in [int(c) for c in args.green_splits.split(",") if c]:
            part = SmPartition(n_exp)
            es, ps = part.first, part.second
            pb_part = prefill_batch(part.sms[1])
            batch = orion.ExpansionBatch(cfg.hq, cfg.hkv, cfg.d, cfg.page, queries, points,
                                         lay.page_table, lay.own_len, policy=args.policy, device=dev,
                                         chunk_tokens=args.chunk, num_sms=part.sms[0], kv_interleaved=args.kv_layout == "interleaved")

            def gstep():
                for l in range(layers):
                    batch.step(q[l], kn[l], vn[l], kc[l], vc[l], out[l], mode=REW, stream=es)

            torch.cuda.synchronize()
            part.sync_before()
            with torch.cuda.stream(es):
                gstep()
            with torch.cuda.stream(ps):
                prefill_layer(pb_part)
            part.synchronize()
            # each alone, in its own partition
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(es)
            for _ in range(steps):
                gstep()
            a1.record(es)
            part.synchronize()
            exp_alone_ms = a0.elapsed_time(a1) / steps
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(ps):
                b0.record(ps)
                for _ in range(10):
                    prefill_layer(pb_part)
                b1.record(ps)
            part.synchronize()
            pf_alone_ms = b0.elapsed_time(b1) / 10
            # together: the prefill partition stays busy for the whole expansion window
            n_pf = int(steps * exp_alone_ms / pf_alone_ms * 1.5) + 4
            s_lo = torch.cuda.Event(enable_timing=True)
            s_hi = torch.cuda.Event(enable_timing=True)
            t_hi = torch.cuda.Event(enable_timing=True)
            pf_ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_pf)]
            with torch.cuda.stream(ps):
                s_lo.record(ps)
                for i in range(n_pf):
                    prefill_layer(pb_part)
                    pf_ev[i].record(ps)
            s_hi.record(es)
            for _ in range(steps):
                gstep()
            t_hi.record(es)
            part.synchronize()
            win = s_hi.elapsed_time(t_hi)
            lag = s_lo.elapsed_time(s_hi)
            done = sum(1 for ev in pf_ev if lag <= s_lo.elapsed_time(ev) <= lag + win)
            exp_tok_s = lay.n_branches * steps / (win / 1e3)
            pf_tflops = done * layer_flop / (win / 1e3) / 1e12
            pf_alone_part = layer_flop / (pf_alone_ms / 1e3) / 1e12
            if pf_alone_part > 1.05 * prefill_alone or done == 0:
                partitioned.append({"expansion_sms": part.sms[0], "prefill_sms": part.sms[1],
                                    "invalid": "prefill GEMMs did not run in this partition "
                                               f"(alone {pf_alone_part:.0f} TFLOP/s, {done} layers in window)"})
                part.close()
                continue
            partitioned.append({
                "expansion_sms": part.sms[0], "prefill_sms": part.sms[1],
                "expansion_alone_in_partition_tok_s": lay.n_branches / (exp_alone_ms / 1e3),
                "prefill_alone_in_partition_tflops": layer_flop / (pf_alone_ms / 1e3) / 1e12,
                "expansion_tok_s": exp_tok_s, "expansion_retained": exp_tok_s / expansion_alone,
                "prefill_tflops": pf_tflops, "prefill_retained": pf_tflops / prefill_alone,
                "sum_retained": exp_tok_s / expansion_alone + pf_tflops / prefill_alone,
                "prefill_layers_in_window": done})
            part.close()
    except Exception as exc:                            # green contexts unavailable: say so
        partitioned = [{"unavailable": f"{type(exc).__name__}: {exc}"}]
    return {"prefill": f"Llama-3-8B layer prefill of {PREFILL_TOKENS} tokens per 'layer': "
                       "[4096x4096]x[4096x{6144,4096,28672}], [4096x14336]x[14336x4096] bf16, "
                       "torch.matmul (cuBLAS), plus the point-prefill attention (orion_point_prefill_attn) "
                       f"of {psub.n_branches} points x Lc {lc} rows ({n_pq} queries), on a low-priority stream",
            "prefill_flop_per_layer": {"gemm": gemm_flop, "point_prefill_attn": attn_flop},
            "expansion": "the headline step on a high-priority stream",
            "prefill_alone_tflops": prefill_alone, "prefill_ms_per_layer": prefill_ms,
            "expansion_alone_tok_s": expansion_alone, "steps": steps, "together": together,
            "partitioned": partitioned,
            "partitioned_note": "green contexts (paper_2510_24390_b200/partition.py): expansion and "
                                "prefill on disjoint SM sets, both launched together; retained = "
                                "rate together / rate alone on the whole GPU"}


def run_e2e(args, batch, layers, q, kn, vn, out, kc, vc, dev, world, total_b):
    """Same step through the public API, inputs from pinned host memory every step and the
    result read back: per layer H2D(q, k_new, v_new) on a copy stream -> append/split/combine
    on the compute stream -> D2H(out) on a third stream, pipelined across layers."""
    import torch
    import torch.distributed as dist
    import paper_2510_24390_b200 as orion
    from paper_2510_24390_b200 import shard
    hq, hkn, hvn = (t.cpu().pin_memory() for t in (q, kn, vn))
    hout = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    comp = torch.cuda.current_stream(dev)
    h2d = torch.cuda.Stream(dev)
    d2h = torch.cuda.Stream(dev)
    in_ready = [torch.cuda.Event() for _ in range(layers)]
    done = [torch.cuda.Event() for _ in range(layers)]
    out_read = [torch.cuda.Event() for _ in range(layers)]
    REW = orion.APPEND_REWRITE

    def step(first):
        for l in range(layers):
            with torch.cuda.stream(h2d):
                if not first:
                    h2d.wait_event(done[l])        # previous step's compute released the inputs
                q[l].copy_(hq[l], non_blocking=True)
                kn[l].copy_(hkn[l], non_blocking=True)
                vn[l].copy_(hvn[l], non_blocking=True)
                in_ready[l].record(h2d)
            comp.wait_event(in_ready[l])
            if not first:
                comp.wait_event(out_read[l])       # previous step's out[l] was read back
            batch.step(q[l], kn[l], vn[l], kc[l], vc[l], out[l], mode=REW)
            done[l].record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done[l])
                hout[l].copy_(out[l], non_blocking=True)
                out_read[l].record(d2h)

    for i in range(max(1, args.warmup)):
        step(i == 0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(args.steps):
        step(False)
    comp.wait_stream(d2h)
    e1.record(comp)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    ms, _ = shard.reduce_timing(ms, 0.0, device=dev)
    ms_step = ms / args.steps
    bi = layers * (q[0].numel() + kn[0].numel() + vn[0].numel()) * 2
    bo = layers * out[0].numel() * 2
    return {"value": total_b / (ms_step / 1e3), "unit": UNIT, "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": bo, "ms_per_step": ms_step,
            "wall_ms_per_step": wall * 1e3 / args.steps,
            "note": "pinned host inputs copied H2D and out copied D2H every step, pipelined per layer"}


def spawn_ranks(args):
    """`--gpus N` without torchrun: launch the N ranks through torch.distributed.run (one process
    per GPU, 127.0.0.1 rendezvous) with the same arguments; rank 0 prints the JSON line."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    global FUSED
    args = parse()
    FUSED = not args.unfused
    cfg = WC.CONFIGS[args.config]
    if args.queries:
        cfg = cfg.with_(n_queries=args.queries)
    layers = args.layers or cfg.layers
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None:
        sys.exit(spawn_ranks(args))
    if world_env is not None and int(world_env) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.impl == "reference":
        run_reference(args, cfg, layers)
    elif args.plan_only:
        plan_only(args, cfg, layers)
    else:
        run_orion(args, cfg, layers)


if __name__ == "__main__":
    main()
