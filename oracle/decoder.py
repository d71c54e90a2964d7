"""O7 — one decoder layer of the expansion decode step, plain NumPy fp64.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product path.

The paper names the models (LLaMA2 7B/13B, Qwen2.5 7B) but no layer internals;
SURVEY.md §8(f) rank 4 fixes a Llama-3-8B-shaped layer with random weights.  Reading M1
(DESIGN.md): the standard pre-norm Llama layer, activations stored in bf16 between ops (fp32
accumulation inside them on the GPU), bf16 KV cache; each op below is computed in fp64 and its
result rounded to bf16 at the same interfaces (`bf16()`), so the comparison isolates the
arithmetic inside each op.  For branch b with residual x_b:

    h   = bf16(RMSNorm(x_b) * w_in)                RMSNorm(x) = x / sqrt(mean(x^2) + eps)
    qkv = bf16(h . W_qkv)                          [Hq*d | Hkv*d | Hkv*d]
    q, k = bf16(RoPE(q, pos_b)), bf16(RoPE(k, pos_b)); v = qkv's V part
    (k, v) appended to b's own run at slot own_len_b (O4), then attention over b's list (O3)
    o   = bf16(bf16(attn) . W_o);  x2 = bf16(x_b + o)
    h2  = bf16(RMSNorm(x2) * w_post); g, u = bf16(h2 . W_gate), bf16(h2 . W_up)
    a   = bf16(SiLU(g) * u);  y = bf16(x2 + bf16(a . W_down))

RoPE (HF `rotate_half` convention, theta = 500000 for Llama-3): for i < d/2 with
f_i = theta^(-2i/d) and angle = pos * f_i: out_i = x_i cos - x_{i+d/2} sin,
out_{i+d/2} = x_{i+d/2} cos + x_i sin.  Reading M2: the position of branch b's new token is its
index in b's concatenated context (its list order, O1/O2), i.e. |ctx(b)| - 1 after the append --
`token_positions` below, computed from O2's bound lists (never from the product).
"""
import numpy as np

from .attention import bf16_to_f64, expand_attn
from .append import kv_append


def bf16(x):
    """Round float64 to the nearest bf16 (ties to even), returned as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32)
    r = np.where(np.isnan(f), np.uint32(0x7FC0), r)
    return (r.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def to_u16(x):
    """float64 values already on the bf16 grid -> raw bf16 bits."""
    return (np.asarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def rmsnorm(x, w, eps=1e-5):
    x = np.asarray(x, dtype=np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * w


def rope(x, pos, theta=500000.0):
    """x [..., H, d], pos [...] (one position per leading index)."""
    d = x.shape[-1]
    half = d // 2
    f = theta ** (-2.0 * np.arange(half) / d)
    ang = np.asarray(pos, dtype=np.float64)[..., None, None] * f      # [..., 1, half]
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def token_positions(bound, slot):
    """Reading M2 -- the position of a branch's new token is its index in the branch's context
    Concat(Prompt_Pre, (+)_k f(k,j), P_j) of Eq. (2), concatenated in list order
    (O1 reading S9): the lengths of its bound segments before OWN (O2 puts OWN last) plus its slot in
    its own run.  bound[b] = [(pages, start, length)] (O2, at the lengths the step starts from);
    slot[b] = the own-run slot the token is written to.  Returns int64 [B]."""
    return np.array([sum(int(n) for (_, _, n) in segs[:-1]) + int(s) for segs, s in zip(bound, slot)],
                    dtype=np.int64)


def silu(x):
    return x / (1.0 + np.exp(-x))


def decoder_layer(x, w, k_cache_u16, v_cache_u16, layout, bound, own_len, pos, hq, hkv, eps=1e-5,
                  theta=500000.0):
    """x [B, hidden] (values on the bf16 grid); w: dict of bf16-grid float64 weights
    (w_in, w_qkv [hidden, (hq+2hkv)d], w_o [hq d, hidden], w_post, w_gate, w_up [hidden, inter],
    w_down [inter, hidden]); bound: O2 segment lists per branch (with the appended token);
    own_len: lengths BEFORE the append; pos [B] RoPE positions.  Returns (y, k_cache, v_cache)."""
    B = x.shape[0]
    d = w["w_o"].shape[0] // hq
    h = bf16(rmsnorm(x, w["w_in"], eps))
    qkv = bf16(h @ w["w_qkv"])
    q = qkv[:, :hq * d].reshape(B, hq, d)
    k = qkv[:, hq * d:(hq + hkv) * d].reshape(B, hkv, d)
    v = qkv[:, (hq + hkv) * d:].reshape(B, hkv, d)
    q = bf16(rope(q, pos, theta))
    k = bf16(rope(k, pos, theta))
    kc, _ = kv_append(k_cache_u16, to_u16(k), layout.page_table, layout.point_pt_off, own_len,
                      layout.page_size)
    vc, _ = kv_append(v_cache_u16, to_u16(v), layout.page_table, layout.point_pt_off, own_len,
                      layout.page_size)
    att, _ = expand_attn(to_u16(q), kc, vc, bound, layout.page_size)
    att = bf16(att).reshape(B, hq * d)
    o = bf16(att @ w["w_o"])
    x2 = bf16(x + o)
    h2 = bf16(rmsnorm(x2, w["w_post"], eps))
    g = bf16(h2 @ w["w_gate"])
    u = bf16(h2 @ w["w_up"])
    a = bf16(silu(g) * u)
    y = bf16(x2 + bf16(a @ w["w_down"]))
    return y, kc, vc
