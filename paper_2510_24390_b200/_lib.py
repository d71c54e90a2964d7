"""ctypes binding of liborion.so (include/orion.h).  Argument marshalling only: every step of
the path (levels, segment lists, binding, planning, append, attention, combine) runs in the
native library.  There is no fallback: a missing or unloadable library raises."""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ORION_LIB overrides the library path (development only, e.g. the ORION_TC_TRACE build
# liborion_trace.so used by tools/trace_tc.sh); the default is the in-tree build.
LIB_PATH = os.environ.get("ORION_LIB") or os.path.join(_HERE, "liborion.so")

OK, ERR_INVALID_ARG, ERR_CYCLE, ERR_UNKNOWN_POINT, ERR_CAPACITY, ERR_UNSUPPORTED, ERR_CUDA = range(7)
EDGE_NULL, EDGE_CONTEXTUAL, EDGE_DEPENDENT = 0, 1, 2
POLICY_ANCESTORS, POLICY_PARENTS_EQ3 = 0, 1
SEG_PREFIX, SEG_CONTENT, SEG_FULL, SEG_OUTPUT, SEG_OWN = range(5)
APPEND_ADVANCE, APPEND_REWRITE = 0, 1

EXPORTED_SYMBOLS = ("orion_dag_waves", "orion_bind_segments", "orion_expand_plan",
                    "orion_plan_get_stats", "orion_kv_append", "orion_expand_attn", "orion_expand_step", "orion_step_launches",
                    "orion_expand_split", "orion_expand_combine", "orion_point_prefill_attn",
                    "orion_expansion_round", "orion_select_branches", "orion_context_base", "orion_rmsnorm",
                    "orion_rope_append", "orion_silu_mul", "orion_last_error", "orion_version")


class Edge(ctypes.Structure):
    _fields_ = [("from_", ctypes.c_int32), ("to", ctypes.c_int32), ("kind", ctypes.c_int32)]


class SegRef(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("point", ctypes.c_int32)]


class Seg(ctypes.Structure):
    _fields_ = [("pt_off", ctypes.c_int32), ("start", ctypes.c_int32), ("len", ctypes.c_int32),
                ("dyn", ctypes.c_int32)]


class AttnShape(ctypes.Structure):
    _fields_ = [("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("page_size", ctypes.c_int32),
                ("sm_scale", ctypes.c_float), ("kv_interleaved", ctypes.c_int32)]


class QueryDesc(ctypes.Structure):
    _fields_ = [("n_points", ctypes.c_int32), ("branch0", ctypes.c_int32),
                ("prefix_pt_off", ctypes.c_int32), ("prefix_len", ctypes.c_int32)]


class PointDesc(ctypes.Structure):
    _fields_ = [("pt_off", ctypes.c_int32), ("content_len", ctypes.c_int32),
                ("capacity", ctypes.c_int32)]


class PlanOpts(ctypes.Structure):
    _fields_ = [("num_sms", ctypes.c_int32), ("chunk_tokens", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("prefill_rows", ctypes.c_int32)]


class PlanStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n_items", "n_pieces", "n_partials", "n_rows",
                                               "unique_tokens", "logical_tokens", "plan_bytes",
                                               "workspace_bytes", "streamed_tokens", "paired", "n_big")]


SEG_DTYPE = np.dtype([("pt_off", np.int32), ("start", np.int32), ("len", np.int32), ("dyn", np.int32)])
SEGREF_DTYPE = np.dtype([("kind", np.int32), ("point", np.int32)])


class OrionError(RuntimeError):
    def __init__(self, code, msg, info=None):
        super().__init__(f"orion status {code}: {msg}")
        self.code = code
        self.info = info


_lib = None


def lib():
    """Load liborion.so once.  Raises (never falls back) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (or `make -C paper_2510_24390_b200/csrc`)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        i32, vp, sz = ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
        L.orion_dag_waves.argtypes = [i32, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, i32]
        L.orion_bind_segments.argtypes = [i32, vp, i32, vp, vp, vp, vp]
        L.orion_expand_plan.argtypes = [P(AttnShape), i32, vp, vp, vp, P(PlanOpts), vp, sz,
                                        P(sz), P(sz)]
        L.orion_plan_get_stats.argtypes = [vp, P(PlanStats)]
        L.orion_kv_append.argtypes = [P(AttnShape), i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, i32, vp]
        L.orion_expand_attn.argtypes = [P(AttnShape), i32, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp,
                                        vp, sz, vp]
        L.orion_expand_split.argtypes = [P(AttnShape), i32, vp, vp, vp, i32, vp, vp, vp, vp, vp,
                                         sz, vp]
        L.orion_expand_combine.argtypes = [P(AttnShape), i32, vp, vp, vp, vp, vp, sz, vp]
        L.orion_point_prefill_attn.argtypes = L.orion_expand_attn.argtypes
        L.orion_step_launches.argtypes = [vp, vp]
        L.orion_expand_step.argtypes = [P(AttnShape), i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, i32,
                                        vp, vp, vp, sz, vp]
        L.orion_expansion_round.argtypes = [i32, vp, vp, vp, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp]
        L.orion_select_branches.argtypes = [i32, vp, vp, vp, i32, vp, vp, vp, i32, vp]
        L.orion_context_base.argtypes = [i32, vp, vp, vp, vp]
        L.orion_rmsnorm.argtypes = [i32, i32, vp, vp, vp, ctypes.c_float, vp, vp, vp]
        L.orion_rope_append.argtypes = [P(AttnShape), i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp,
                                        ctypes.c_float, i32, vp]
        L.orion_silu_mul.argtypes = [i32, i32, vp, vp, vp]
        for f in ("orion_expand_split", "orion_expand_combine", "orion_dag_waves", "orion_bind_segments", "orion_expand_plan",
                  "orion_plan_get_stats", "orion_kv_append", "orion_expand_attn", "orion_point_prefill_attn",
                  "orion_expand_step", "orion_step_launches", "orion_expansion_round", "orion_select_branches", "orion_context_base", "orion_rmsnorm",
                  "orion_rope_append", "orion_silu_mul"):
            getattr(L, f).restype = ctypes.c_int32
        L.orion_last_error.restype = ctypes.c_char_p
        L.orion_last_error.argtypes = []
        L.orion_version.restype = ctypes.c_char_p
        L.orion_version.argtypes = []
        _lib = L
    return _lib


def check(code, info=None):
    if code != OK:
        raise OrionError(code, lib().orion_last_error().decode(), info)


def ptr(a):
    """Address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return a.data_ptr()


def aligned_empty(nbytes, align=64):
    """A zeroed uint8 numpy buffer whose data pointer is `align`-byte aligned."""
    raw = np.zeros(nbytes + align, dtype=np.uint8)
    off = (-raw.ctypes.data) % align
    return raw[off:off + nbytes]
