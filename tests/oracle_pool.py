"""Runs the (slow, single-threaded) oracle O3 over many branches in parallel worker processes, for
the full-size GPU parity tests (c4, c5).  Test infrastructure only; the oracle itself is unchanged:
each worker calls oracle.step.expand_step on a contiguous block of branches, on the same bytes
(the caches are shared through memory-mapped .npy files, never pickled), and the blocks are
concatenated in branch order."""
import multiprocessing as mp
import os
import tempfile

import numpy as np


def _work(args):
    fn, lay, paths, policy, branches, own_len, scale = args
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    from oracle import step as OS, prefill as OP
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)                              # one BLAS thread per worker process
    q, k, v = (np.load(p, mmap_mode="r") for p in paths)
    f = OS.expand_step if fn == "decode" else OP.point_prefill
    return f(lay, np.asarray(q), k, v, policy=policy, branches=branches, own_len=own_len, scale=scale)


def expand_step_parallel(lay, q_u16, k_u16, v_u16, policy=0, branches=None, own_len=None, scale=None,
                         workers=None):
    """oracle.step.expand_step(lay, q, k, v, policy, branches, own_len) computed by `workers`
    spawned processes (default: the usable cores, at most 32)."""
    return _parallel("decode", lay, q_u16, k_u16, v_u16, policy, branches, own_len, scale, workers)


def point_prefill_parallel(lay, q_u16, k_u16, v_u16, policy=0, branches=None, own_len=None, scale=None,
                           workers=None):
    """oracle.prefill.point_prefill(...) in worker processes (as expand_step_parallel)."""
    return _parallel("prefill", lay, q_u16, k_u16, v_u16, policy, branches, own_len, scale, workers)


def _parallel(fn, lay, q_u16, k_u16, v_u16, policy, branches, own_len, scale, workers):
    if branches is None:
        branches = list(range(lay.n_branches))
    branches = list(branches)
    workers = workers or min(32, len(os.sched_getaffinity(0)))
    workers = max(1, min(workers, len(branches)))
    base = "/dev/shm" if os.path.isdir("/dev/shm") else None
    with tempfile.TemporaryDirectory(dir=base) as d:
        paths = []
        for name, a in (("q", q_u16), ("k", k_u16), ("v", v_u16)):
            p = os.path.join(d, name + ".npy")
            np.save(p, np.ascontiguousarray(a))
            paths.append(p)
        # interleaved blocks balance long and short contexts across workers
        chunks = [branches[i::workers] for i in range(workers)]
        ctx = mp.get_context("spawn")
        keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
        saved = {k: os.environ.get(k) for k in keys}
        os.environ.update({k: "1" for k in keys})     # inherited by the spawned workers
        try:
            with ctx.Pool(workers) as pool:
                res = pool.map(_work, [(fn, lay, paths, policy, c, own_len, scale) for c in chunks])
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    n = len(branches)
    out = np.zeros((n,) + res[0][0].shape[1:])
    lse = np.zeros((n,) + res[0][1].shape[1:])
    for i, (o, l) in enumerate(res):
        out[i::workers] = o
        lse[i::workers] = l
    return out, lse
