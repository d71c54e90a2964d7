"""SM partitioning for co-scheduling (decode is memory-
bound, prefill compute-bound, so running them side by side on disjoint SM sets lets each use the
hardware the other leaves idle).  Stream priorities cannot do this on their own: a persistent
kernel's CTAs, or cuBLAS's, are never preempted, so two streams mostly time-slice (bench
`prefill_costream`).  A green context owns a fixed set of SMs; work launched on a green context's
stream -- the orion kernels through the C ABI, or torch / cuBLAS through torch.cuda.ExternalStream
-- runs only on those SMs.

The orion split kernels are persistent (one CTA per SM): give them a plan built with
`num_sms` = the partition's SM count, so the grid fits the partition.

Streams of different contexts are not ordered with each other: make a green stream wait for
inputs produced elsewhere (`sync_before`) and synchronise green streams explicitly.
"""
import torch


def _check(res):
    err = res[0] if isinstance(res, tuple) else res
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver call failed: {err}")
    if isinstance(res, tuple):
        return res[1] if len(res) == 2 else res[1:]
    return None


class SmPartition:
    """Two green contexts on one device: `first` with (at least) n_first SMs, `second` with the
    rest.  Attributes: streams (torch.cuda.ExternalStream) and SM counts of both."""

    def __init__(self, n_first, device=0, priority_first=0, priority_second=0):
        import cuda.bindings.driver as d
        self._d = d
        torch.zeros(1, device=f"cuda:{device}")          # primary context exists
        dev = _check(d.cuDeviceGet(device))
        res = _check(d.cuDeviceGetDevResource(dev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
        self.total_sms = int(res.sm.smCount)
        groups, _, rem = _check(d.cuDevSmResourceSplitByCount(1, res, 0, int(n_first)))
        self._ctx = []
        self.streams = []
        self.sms = []
        for r, prio in ((groups[0], priority_first), (rem, priority_second)):
            desc = _check(d.cuDevResourceGenerateDesc([r], 1))
            g = _check(d.cuGreenCtxCreate(desc, dev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
            st = _check(d.cuGreenCtxStreamCreate(g, d.CUstream_flags.CU_STREAM_NON_BLOCKING, prio))
            self._ctx.append(g)
            self.streams.append(torch.cuda.ExternalStream(int(st)))
            self.sms.append(int(r.sm.smCount))

    @property
    def first(self):
        return self.streams[0]

    @property
    def second(self):
        return self.streams[1]

    def sync_before(self, src_stream=None):
        """Make both partition streams wait for the work queued so far on src_stream (default:
        torch's current stream)."""
        ev = torch.cuda.Event()
        ev.record(src_stream or torch.cuda.current_stream())
        for s in self.streams:
            s.wait_event(ev)

    def synchronize(self):
        for s in self.streams:
            s.synchronize()

    def close(self):
        for g in self._ctx:
            self._d.cuGreenCtxDestroy(g)
        self._ctx = []
