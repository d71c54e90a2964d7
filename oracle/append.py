"""O4 — KV append of the decode step (reading S15: append, then attend).

For every branch b and kv head g, the new token's K (and V) row is written to
token position own_len[b] of b's own segment:
    cache[page_table[own_pt_off[b] + own_len[b] // P], g, own_len[b] % P, :] = k_new[b, g, :]
then own_len[b] += 1.  Bit-exact copy (no arithmetic on the values).
Rewrite mode (bench steady state): write position own_len[b] - 1, no increment.
"""
import numpy as np


def kv_append(cache_u16, new_u16, page_table, own_pt_off, own_len, page_size, rewrite=False):
    cache = np.array(cache_u16, copy=True)
    own = np.array(own_len, dtype=np.int64, copy=True)
    B, Hkv, _ = new_u16.shape
    for b in range(B):
        pos = own[b] - 1 if rewrite else own[b]
        page = page_table[own_pt_off[b] + pos // page_size]
        for g in range(Hkv):
            cache[page, g, pos % page_size, :] = new_u16[b, g, :]
        if not rewrite:
            own[b] += 1
    return cache, own
