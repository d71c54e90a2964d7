"""Pins for oracle O7 (decoder layer): an independent implementation --
Hugging Face transformers' LlamaDecoderLayer in fp64 -- on a causal sequence whose prefix K/V
seed the paged cache, agreeing with O7 within the bf16 rounding of its interfaces; torch's own
bf16 conversion; RoPE against its complex-multiplication form and the relative-position
property; closed forms of RMSNorm / SiLU; the residual identity of a layer with zero outputs."""
import numpy as np
import pytest
import torch

from oracle import decoder as DE, step as OS
from workloads import configs as C, tensors as T, dags as W


def test_bf16_matches_torch_conversion():
    x = np.random.default_rng(1).standard_normal(100000) * np.logspace(-3, 3, 100000)
    want = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(DE.bf16(x), want)


def test_rope_complex_form_and_relative_position():
    rng = np.random.default_rng(2)
    d, H = 64, 3
    x = rng.standard_normal((5, H, d))
    pos = np.array([0, 1, 7, 100, 4097])
    out = DE.rope(x, pos, theta=10000.0)
    # complex form: (x_i + i x_{i+d/2}) * exp(i pos f_i)
    z = x[..., :d // 2] + 1j * x[..., d // 2:]
    f = 10000.0 ** (-2.0 * np.arange(d // 2) / d)
    zr = z * np.exp(1j * pos[:, None, None] * f)
    assert np.allclose(out, np.concatenate([zr.real, zr.imag], -1), atol=1e-12)
    assert np.allclose(out[0], x[0])                                # position 0: identity
    # q(m).k(n) depends on m - n only
    q, k = rng.standard_normal((1, 1, d)), rng.standard_normal((1, 1, d))
    a = (DE.rope(q, [37]) * DE.rope(k, [30])).sum()
    b = (DE.rope(q, [7]) * DE.rope(k, [0])).sum()
    assert abs(a - b) < 1e-9


def test_rmsnorm_and_silu_closed_forms():
    x = np.full((2, 8), 3.0)
    assert np.allclose(DE.rmsnorm(x, 2.0, eps=0.0), 2.0)
    assert DE.silu(np.array([0.0]))[0] == 0.0
    assert np.allclose(DE.silu(np.array([30.0])), 30.0, rtol=1e-12)
    from scipy.special import expit
    v = np.linspace(-6, 6, 101)
    assert np.allclose(DE.silu(v), v * expit(v), atol=1e-14)


def small_model(rng, hidden=128, hq=4, hkv=2, d=32, inter=192, scale=0.08):
    g = lambda *s: DE.bf16(rng.standard_normal(s) * scale)
    return dict(w_in=DE.bf16(1 + 0.1 * rng.standard_normal(hidden)), w_qkv=g(hidden, (hq + 2 * hkv) * d),
                w_o=g(hq * d, hidden), w_post=DE.bf16(1 + 0.1 * rng.standard_normal(hidden)),
                w_gate=g(hidden, inter), w_up=g(hidden, inter), w_down=g(inter, hidden))


def test_matches_hf_llama_decoder_layer():
    # One causal sequence: HF computes the whole sequence in fp64; its (RoPE'd) K/V of tokens
    # 0..L-2 seed a paged cache, and O7 decodes token L-1 (a single branch whose list is the
    # prefix + its own run).  Differences come from O7's bf16 interfaces only.
    from transformers import LlamaConfig
    from transformers.models.llama.modeling_llama import LlamaDecoderLayer, LlamaRotaryEmbedding
    from transformers.cache_utils import DynamicCache
    rng = np.random.default_rng(3)
    hidden, hq, hkv, d, inter, L = 128, 4, 2, 32, 192, 40
    w = small_model(rng, hidden, hq, hkv, d, inter)
    cfg = LlamaConfig(hidden_size=hidden, intermediate_size=inter, num_attention_heads=hq,
                      num_key_value_heads=hkv, head_dim=d, rms_norm_eps=1e-5, rope_theta=500000.0,
                      hidden_act="silu", attention_bias=False, mlp_bias=False,
                      max_position_embeddings=4096)
    cfg._attn_implementation = "eager"
    layer = LlamaDecoderLayer(cfg, 0).double().eval()
    sd = {"input_layernorm.weight": w["w_in"], "post_attention_layernorm.weight": w["w_post"],
          "self_attn.q_proj.weight": w["w_qkv"][:, :hq * d].T,
          "self_attn.k_proj.weight": w["w_qkv"][:, hq * d:(hq + hkv) * d].T,
          "self_attn.v_proj.weight": w["w_qkv"][:, (hq + hkv) * d:].T,
          "self_attn.o_proj.weight": w["w_o"].T, "mlp.gate_proj.weight": w["w_gate"].T,
          "mlp.up_proj.weight": w["w_up"].T, "mlp.down_proj.weight": w["w_down"].T}
    layer.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()})
    rot = LlamaRotaryEmbedding(cfg).double()
    x = DE.bf16(rng.standard_normal((1, L, hidden)))
    xt = torch.from_numpy(x)
    pos = torch.arange(L)[None]
    cos, sin = rot(xt, pos)
    mask = torch.full((L, L), float("-inf"), dtype=torch.float64).triu(1)[None, None]
    cache = DynamicCache()
    with torch.no_grad():
        y_hf = layer(xt, attention_mask=mask, position_ids=pos, past_key_values=cache, use_cache=True,
                     position_embeddings=(cos, sin))
    y_hf = (y_hf[0] if isinstance(y_hf, tuple) else y_hf)[0, -1].numpy()
    k_all = cache.layers[0].keys[0].numpy()                          # [hkv, L, d] after RoPE
    v_all = cache.layers[0].values[0].numpy()
    # paged cache: prefix run = tokens 0..L-2, the branch's own run receives token L-1 (append)
    page = 16
    ccfg = C.CONFIGS["c1"].with_(hq=hq, hkv=hkv, d=d, page=page, lp=L - 1, t=page, lc=0, n_queries=1)
    lay = T.make_layout(ccfg, dag_override=lambda: W.wide(1))
    lay.own_len[:] = 0
    kc = np.zeros((lay.num_pages, hkv, page, d), np.uint16)
    vc = np.zeros_like(kc)
    pages = lay.pages_of(lay.prefix_pt_off[0], L - 1)
    for t in range(L - 1):
        kc[pages[t // page], :, t % page] = DE.to_u16(DE.bf16(k_all[:, t]))
        vc[pages[t // page], :, t % page] = DE.to_u16(DE.bf16(v_all[:, t]))
    own_after = lay.own_len + 1
    bound = OS.bound_segments(lay, own_len=own_after)
    y, _, _ = DE.decoder_layer(x[0, -1:], w, kc, vc, lay, bound, lay.own_len, np.array([L - 1]), hq, hkv)
    err = np.abs(y[0] - y_hf)
    assert err.max() < 0.06 and np.linalg.norm(y[0] - y_hf) / np.linalg.norm(y_hf) < 1e-2, err.max()


def test_zero_output_projections_leave_the_residual():
    rng = np.random.default_rng(4)
    w = small_model(rng)
    w["w_o"][:] = 0.0
    w["w_down"][:] = 0.0
    cfg = C.CONFIGS["c1"].with_(hq=4, hkv=2, d=32, page=16, lp=20, t=16, lc=4, n_queries=1)
    lay = T.make_layout(cfg, dag_override=W.fig4)
    kc = T.bf16_randn_u16((lay.num_pages, 2, 16, 32), 1)
    kc = kc.view(torch.int16).numpy().view(np.uint16)
    vc = kc.copy()
    own = lay.own_len - 1
    x = DE.bf16(rng.standard_normal((lay.n_branches, 128)))
    y, _, _ = DE.decoder_layer(x, w, kc, vc, lay, OS.bound_segments(lay), own, own + 20, 4, 2)
    assert np.array_equal(y, x)


# ---- reading M2: the RoPE position of a branch's token, derived from O1/O2 (not the product)
def test_token_positions_closed_forms():
    """Dependent chain (ANCESTORS: [PREFIX, FULL(1..j-1), OWN(j)]): branch j's token sits where
    ordinary causal decode of [prefix | S_1 | ... | S_j] puts it, Lp + sum_{k<j} |S_k| + slot.
    Wide (edgeless): Lp + slot.  Diamond under PARENTS_EQ3: point 4 reads [PREFIX, OUTPUT(2),
    OUTPUT(3), OWN(4)] (Eq. (3) f = Output_k), so Lp + (|S_2| - Lc) + (|S_3| - Lc) +
    slot; under ANCESTORS [PREFIX, CONTENT(1), FULL(2), FULL(3), OWN(4)]: Lp + Lc + |S_2| + |S_3|."""
    from oracle import dag as OD
    cfg = C.CONFIGS["c1"].with_(page=16, lp=37, t=40, lc=8, n_queries=2)
    lay = T.make_layout(cfg, ragged=True, extra_tokens=16, dag_override=lambda: W.chain(6))
    for slot in (lay.own_len.copy(), lay.own_len - 1):
        pos = DE.token_positions(OS.bound_segments(lay, own_len=lay.own_len), slot)
        for qi in range(2):
            b0 = int(lay.branch0[qi])
            for j in range(6):
                want = int(lay.prefix_len[qi]) + int(lay.own_len[b0:b0 + j].sum()) + int(slot[b0 + j])
                assert pos[b0 + j] == want
    lay = T.make_layout(cfg, ragged=True, extra_tokens=16, dag_override=lambda: W.wide(5))
    pos = DE.token_positions(OS.bound_segments(lay), lay.own_len)
    assert np.array_equal(pos, lay.prefix_len[lay.branch_query] + lay.own_len)
    lay = T.make_layout(cfg.with_(n_queries=1), ragged=True, extra_tokens=16, dag_override=W.diamond)
    o = lay.own_len
    pos = DE.token_positions(OS.bound_segments(lay, OD.PARENTS_EQ3), o)
    assert pos[3] == 37 + (o[1] - 8) + (o[2] - 8) + o[3]
    pos = DE.token_positions(OS.bound_segments(lay, OD.ANCESTORS), o)
    assert pos[3] == 37 + 8 + o[1] + o[2] + o[3]
    assert pos[1] == 37 + 8 + o[1] and pos[0] == 37 + o[0]


def _hf_layer(w, hidden, hq, hkv, d, inter):
    from transformers import LlamaConfig
    from transformers.models.llama.modeling_llama import LlamaDecoderLayer, LlamaRotaryEmbedding
    cfg = LlamaConfig(hidden_size=hidden, intermediate_size=inter, num_attention_heads=hq,
                      num_key_value_heads=hkv, head_dim=d, rms_norm_eps=1e-5, rope_theta=500000.0,
                      hidden_act="silu", attention_bias=False, mlp_bias=False,
                      max_position_embeddings=4096)
    cfg._attn_implementation = "eager"
    layer = LlamaDecoderLayer(cfg, 0).double().eval()
    sd = {"input_layernorm.weight": w["w_in"], "post_attention_layernorm.weight": w["w_post"],
          "self_attn.q_proj.weight": w["w_qkv"][:, :hq * d].T,
          "self_attn.k_proj.weight": w["w_qkv"][:, hq * d:(hq + hkv) * d].T,
          "self_attn.v_proj.weight": w["w_qkv"][:, (hq + hkv) * d:].T,
          "self_attn.o_proj.weight": w["w_o"].T, "mlp.gate_proj.weight": w["w_gate"].T,
          "mlp.up_proj.weight": w["w_up"].T, "mlp.down_proj.weight": w["w_down"].T}
    layer.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()})
    return layer, LlamaRotaryEmbedding(cfg).double()


def test_chain_positions_match_hf_causal_decode():
    """A 2-point Dependent chain is ordinary causal decode of [prefix | S_1 | S_2] (north_star;
    reading S6/S7): HF's LlamaDecoderLayer over that sequence in fp64 gives the last token's output;
    O7 decodes the same token as branch 2 of the chain, its K/V history in three page runs, with the
    positions from token_positions.  Mutations of the position rule (dropping FULL(1), counting the
    own run twice) fail the same gate."""
    from transformers.cache_utils import DynamicCache
    rng = np.random.default_rng(11)
    hidden, hq, hkv, d, inter = 128, 4, 2, 32, 192
    Lp, T1, T2, page = 21, 30, 13, 16
    L = Lp + T1 + T2
    w = small_model(rng, hidden, hq, hkv, d, inter)
    w["w_qkv"] = DE.bf16(rng.standard_normal(w["w_qkv"].shape) * 0.2)   # sharp, position-sensitive attention
    layer, rot = _hf_layer(w, hidden, hq, hkv, d, inter)
    x = DE.bf16(rng.standard_normal((1, L, hidden)))
    xt = torch.from_numpy(x)
    p = torch.arange(L)[None]
    cos, sin = rot(xt, p)
    mask = torch.full((L, L), float("-inf"), dtype=torch.float64).triu(1)[None, None]
    cache = DynamicCache()
    with torch.no_grad():
        y_hf = layer(xt, attention_mask=mask, position_ids=p, past_key_values=cache, use_cache=True,
                     position_embeddings=(cos, sin))
    y_hf = (y_hf[0] if isinstance(y_hf, tuple) else y_hf)[0, -1].numpy()
    k_all = cache.layers[0].keys[0].numpy()
    v_all = cache.layers[0].values[0].numpy()
    ccfg = C.CONFIGS["c1"].with_(hq=hq, hkv=hkv, d=d, page=page, lp=Lp, t=max(T1, T2), lc=4, n_queries=1)
    lay = T.make_layout(ccfg, extra_tokens=page, dag_override=lambda: W.chain(2))
    kc = np.zeros((lay.num_pages, hkv, page, d), np.uint16)
    vc = np.zeros_like(kc)
    runs = [(lay.pages_of(lay.prefix_pt_off[0], Lp), 0, Lp),
            (lay.pages_of(lay.point_pt_off[0], T1), Lp, T1),
            (lay.pages_of(lay.point_pt_off[1], T2), Lp + T1, T2 - 1)]
    for pages, t0, n in runs:
        for t in range(n):
            kc[pages[t // page], :, t % page] = DE.to_u16(DE.bf16(k_all[:, t0 + t]))
            vc[pages[t // page], :, t % page] = DE.to_u16(DE.bf16(v_all[:, t0 + t]))
    own = np.array([T1, T2 - 1])                       # lengths the step starts from
    pos = DE.token_positions(OS.bound_segments(lay, own_len=own), own)
    assert pos[1] == L - 1
    bound = OS.bound_segments(lay, own_len=np.array([T1, T2]))   # branch 2 after its append
    xin = np.stack([x[0, -2], x[0, -1]])

    def err(pp):
        y, _, _ = DE.decoder_layer(xin, w, kc, vc, lay, bound, own, pp, hq, hkv)
        return np.linalg.norm(y[1] - y_hf) / np.linalg.norm(y_hf)

    assert err(pos) < 1.5e-2                            # bf16 interface rounding only
    assert err(pos - np.array([0, T1])) > 0.1          # FULL(1) dropped from the base
    assert err(pos + own) > 0.1                         # own run counted twice
    assert err(pos - 1) > 0.1                           # off by one
