"""Test-side helpers for pinning the oracle: an independent contiguous view of a paged
segment (page blocks concatenated, not token-by-token gather) and fp64 SDPA."""
import numpy as np
import torch


def u16(t):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def f64(t):
    """bf16 torch tensor -> float64 torch tensor (torch's own widening)."""
    return t.to(torch.float64)


def contiguous(cache_bf16, page_table, pt_off, n_tokens, page_size):
    """[n_tokens, Hkv, d] float64 view of a page run: whole pages concatenated, then truncated."""
    n_pages = -(-n_tokens // page_size)
    blocks = [cache_bf16[int(page_table[pt_off + i])].permute(1, 0, 2) for i in range(n_pages)]
    if not blocks:
        return torch.zeros(0, cache_bf16.shape[1], cache_bf16.shape[3], dtype=torch.float64)
    return torch.cat(blocks, 0)[:n_tokens].to(torch.float64)


def sdpa_decode(q_row_heads, k_seq, v_seq, scale=None):
    """q [Hq, d]; k/v [n, Hkv, d] -> out [Hq, d] via torch SDPA (fp64, CPU) with repeat_kv GQA."""
    hq, d = q_row_heads.shape
    hkv = k_seq.shape[1]
    g = hq // hkv
    k = k_seq.permute(1, 0, 2).repeat_interleave(g, dim=0)   # [Hq, n, d]
    v = v_seq.permute(1, 0, 2).repeat_interleave(g, dim=0)
    q = q_row_heads[:, None, :]                               # [Hq, 1, d]
    out = torch.nn.functional.scaled_dot_product_attention(q, k, v, scale=scale)
    return out[:, 0, :]
