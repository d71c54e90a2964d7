"""N>1 host path on CPU: query sharding, per-rank plans and the max/sum timing reductions over a
real torch.distributed process group (gloo, world_size 2, 127.0.0.1).  The data path has no
collective; the GPU-side check that a rank's outputs equal the single-GPU ones
bitwise is tests/test_gpu_parity.py::test_strong_shards_bitwise."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_24390_b200 import shard  # noqa: E402
from workloads import configs as C, tensors as T  # noqa: E402


def test_partition_equal_costs_contiguous_blocks():
    for q, n in [(64, 8), (64, 3), (5, 8), (1, 2), (0, 4)]:
        parts = shard.partition_queries([1.0] * q, n)
        assert len(parts) == n
        assert sum(parts, []) == list(range(q))              # contiguous, in order, exactly once
        for r, p in enumerate(parts):
            assert p == [i for i in range(q) if (i * n) // q == r]
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1


def test_partition_lpt_unequal_costs():
    rng = np.random.default_rng(3)
    for trial in range(20):
        q, n = int(rng.integers(1, 40)), int(rng.integers(1, 6))
        costs = rng.integers(1, 100, q).astype(float)
        parts = shard.partition_queries(costs, n)
        assert sorted(sum(parts, [])) == list(range(q))
        loads = [costs[p].sum() if p else 0.0 for p in parts]
        # LPT bound: the most loaded rank exceeds the mean by at most the largest single cost
        assert max(loads) <= costs.sum() / n + costs.max() + 1e-9
        assert all(p == sorted(p) for p in parts)
    # ties broken by query id: equal-cost pairs go to ranks in id order
    assert shard.partition_queries([5, 5, 1, 1], 2) == [[0, 2], [1, 3]]


def test_rank_queries_modes_and_errors():
    assert shard.rank_queries(10, 1, 4, "weak") == list(range(10))
    assert shard.rank_queries(10, 3, 4, "strong") == [8, 9]
    assert shard.rank_queries(10, 0, 1, "strong") == list(range(10))
    with pytest.raises(ValueError):
        shard.rank_queries(10, 4, 4)
    with pytest.raises(ValueError):
        shard.rank_queries(10, 0, 2, "diagonal")
    assert shard.rank_seed(7, 0) != shard.rank_seed(7, 1)
    assert shard.reduce_timing(3.5, 12) == (3.5, 12.0)       # no process group: identity


def test_subset_layout_keeps_query_data():
    cfg = C.CONFIGS["c3"]
    lay = T.make_layout(cfg, ragged=True)
    qs = shard.rank_queries(cfg.n_queries, 1, 2, "strong")
    sub, br = T.subset_layout(lay, qs)
    assert sub.n_queries == len(qs) and sub.n_branches == len(br)
    for i, q in enumerate(qs):
        b0, n = int(lay.branch0[q]), int(lay.n_points[q])
        assert list(br[sub.branch0[i]:sub.branch0[i] + n]) == list(range(b0, b0 + n))
        assert sub.prefix_pt_off[i] == lay.prefix_pt_off[q] and sub.edges[i] == lay.edges[q]
    assert np.array_equal(sub.point_pt_off, lay.point_pt_off[br])
    assert np.array_equal(sub.own_len, lay.own_len[br])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, scaling, results):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from tests.test_host_lib import _bind_layout
    import paper_2510_24390_b200 as orion
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = C.CONFIGS["c3"]
        qs = shard.rank_queries(cfg.n_queries, rank, world, scaling)
        full = T.make_layout(cfg, seed=shard.rank_seed(cfg.seed, rank) if scaling == "weak" else cfg.seed)
        lay, br = T.subset_layout(full, qs)
        offs, segs = _bind_layout(cfg, lay, 0)
        plan, ws = orion.expand_plan(cfg.hq, cfg.hkv, cfg.d, cfg.page, offs, segs, lay.own_len)
        st = orion.plan_stats(plan)
        # this rank's plan covers exactly its branches' rows
        assert st["n_rows"] == lay.n_branches * cfg.hq
        ms, units = shard.reduce_timing(10.0 + rank, float(lay.n_branches))
        got = [None] * world
        dist.all_gather_object(got, (qs, [int(b) for b in br]))
        results[rank] = (ms, units, got, st["unique_tokens"])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_two_rank_gloo(scaling):
    world = 2
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), scaling, results), nprocs=world,
                       join=True, start_method="spawn")
    cfg = C.CONFIGS["c3"]
    lay = T.make_layout(cfg)
    for rank in range(world):
        ms, units, got, _ = results[rank]
        assert ms == 10.0 + world - 1                         # max over ranks
        shards = [g[0] for g in got]
        if scaling == "strong":
            assert sorted(sum(shards, [])) == list(range(cfg.n_queries))   # a partition
            assert units == lay.n_branches                    # sum over ranks = whole batch
            assert sorted(sum([g[1] for g in got], [])) == list(range(lay.n_branches))
        else:
            assert all(s == list(range(cfg.n_queries)) for s in shards)
            assert units == world * lay.n_branches


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_bench_launcher_two_ranks_plan_only(scaling):
    """bench.py's own N>1 path on CPU: `--gpus 2` without torchrun launches the two ranks itself
    (torch.distributed.run, 127.0.0.1, gloo under --plan-only), each shards / plans its queries, and
    rank 0 prints one JSON line with the whole-job branch count and every rank's share."""
    import json
    import subprocess
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plan-only",
                        "--config", "c3", "--scaling", scaling], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    cfg = C.CONFIGS["c3"]
    lay = T.make_layout(cfg)
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["plan_only"]
    qs = [p["queries"] for p in sorted(d["per_rank"], key=lambda p: p["rank"])]
    if scaling == "strong":
        assert qs == shard.partition_queries([1.0] * cfg.n_queries, 2)
        assert d["config"]["branches_per_step"] == lay.n_branches
    else:
        assert qs == [list(range(cfg.n_queries))] * 2
        assert d["config"]["branches_per_step"] == 2 * lay.n_branches


def test_bench_rejects_inconsistent_world():
    import subprocess
    env = dict(os.environ, WORLD_SIZE="3", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plan-only"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=3" in r.stderr
