"""O3 — the attention of one expansion decode step, by its plain definition (NumPy fp64).

For every branch b and query head h (kv head g = h // G, reading S16):
    ctx(b)   = concatenation of b's bound segments, IN LIST ORDER            (Eq. (2) Concat)
    s        = scale * q[b,h] . K_ctx^T                                       (scale = 1/sqrt(d))
    out[b,h] = softmax(s) . V_ctx ,   lse[b,h] = m + ln(sum exp(s - m))
bf16 inputs are widened exactly: (u16 << 16) viewed as float32, then float64.

O3' (`masked_pool_attn`) is a second, independent formulation for tiny configs:
the query's whole token pool with a 0/1 mask, used to pin the binding logic.
"""
import numpy as np


def bf16_to_f64(u16):
    """Exact widening of raw bf16 bits (uint16 array) to float64."""
    u = np.left_shift(np.asarray(u16, dtype=np.uint16), 16, dtype=np.uint32)
    return u.view(np.float32).astype(np.float64)


def gather_tokens(cache, pages, start, length, g, page_size):
    """Rows [start, start+length) of the segment whose t-th token is on page pages[t // P], row
    t % P: the pages covering the range, read whole in order, then the range cut out of them."""
    if length <= 0:
        return cache[:0, g, 0]
    p0, p1 = start // page_size, (start + length - 1) // page_size + 1
    blk = cache[np.asarray(pages, dtype=np.int64)[p0:p1], g].reshape(-1, cache.shape[-1])
    off = start - p0 * page_size
    return blk[off:off + length]


def context(cache, segs, g, page_size):
    """K_ctx (or V_ctx) of one branch and kv head: its segments concatenated in list order."""
    parts = [gather_tokens(cache, pages, s, n, g, page_size) for (pages, s, n) in segs]
    return np.concatenate(parts, axis=0)


def attend(q_rows, k_ctx, v_ctx, scale):
    """softmax(scale q K^T) V for a block of query rows; returns (out, lse)."""
    s = scale * (q_rows @ k_ctx.T)
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    l = p.sum(axis=1, keepdims=True)
    out = (p @ v_ctx) / l
    lse = (m + np.log(l))[:, 0]
    return out, lse


def expand_attn(q_u16, k_u16, v_u16, bound, page_size, scale=None):
    """q_u16 [B,Hq,d], k/v_u16 [pages,Hkv,P,d] (raw bf16 bits); bound[b] = [(pages,start,len)].
    Returns out [B,Hq,d] float64 and lse [B,Hq] float64."""
    q = bf16_to_f64(q_u16)
    B, Hq, d = q.shape
    Hkv = k_u16.shape[1]
    G = Hq // Hkv
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    out = np.zeros((B, Hq, d))
    lse = np.zeros((B, Hq))
    for b in range(B):
        for g in range(Hkv):
            # gather the raw bf16 rows, then widen them exactly (the same values as widening the
            # whole cache first, without materialising an fp64 copy of it)
            kc = bf16_to_f64(context(k_u16, bound[b], g, page_size))
            vc = bf16_to_f64(context(v_u16, bound[b], g, page_size))
            o, l = attend(q[b, g * G:(g + 1) * G], kc, vc, scale)
            out[b, g * G:(g + 1) * G] = o
            lse[b, g * G:(g + 1) * G] = l
    return out, lse


def masked_pool_attn(q_u16, k_u16, v_u16, pool, mask, page_size, scale=None):
    """O3': pool = list of (page, row) token locations of the whole query; mask[b, t] in {0,1}.
    Dense masked softmax over the pool (fp64)."""
    q = bf16_to_f64(q_u16)
    k = bf16_to_f64(k_u16)
    v = bf16_to_f64(v_u16)
    B, Hq, d = q.shape
    Hkv = k.shape[1]
    G = Hq // Hkv
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    out = np.zeros((B, Hq, d))
    lse = np.zeros((B, Hq))
    mask = np.asarray(mask, dtype=bool)
    for g in range(Hkv):
        kp = np.stack([k[p, g, r] for (p, r) in pool])
        vp = np.stack([v[p, g, r] for (p, r) in pool])
        for b in range(B):
            for h in range(g * G, (g + 1) * G):
                s = scale * (kp @ q[b, h])
                s = np.where(mask[b], s, -np.inf)
                m = s.max()
                p = np.where(mask[b], np.exp(s - m), 0.0)
                out[b, h] = (p @ vp) / p.sum()
                lse[b, h] = m + np.log(p.sum())
    return out, lse
