"""A decoder model around the expansion attention (oracle O7): Llama-3-8B-
shaped layers (pre-norm RMSNorm, GQA attention with RoPE, SwiGLU MLP) with random weights, so the
whole-model expansion step can be measured in the paper's unit (generated tokens / s).

Per layer: orion_rmsnorm (fused with the previous residual add) -> QKV GEMM -> orion_rope_append
(RoPE fused into the KV append) -> the expansion attention (orion_expand_attn) -> O GEMM ->
orion_rmsnorm (fused residual add) -> gate|up GEMM -> orion_silu_mul -> down GEMM; the last
residual add is fused into the next layer's norm.  The GEMMs are plain library calls
(torch.matmul -> cuBLAS, bf16 in / bf16 out, fp32 accumulation); every other step is an orion
kernel through the C ABI.  Activations are bf16 between steps (reading M1).
"""
import math

import torch

from . import APPEND_ADVANCE, APPEND_REWRITE, rmsnorm, silu_mul


class DecoderModel:
    def __init__(self, n_layers, hidden=4096, hq=32, hkv=8, d=128, inter=14336, rope_theta=500000.0,
                 eps=1e-5, device="cuda", seed=0, init_scale=1.0):
        self.n_layers, self.hidden, self.hq, self.hkv, self.d, self.inter = n_layers, hidden, hq, hkv, d, inter
        self.theta, self.eps = rope_theta, eps
        dev = torch.device(device)
        g = torch.Generator(device=dev)
        g.manual_seed(seed)

        def mat(k, n):
            w = torch.randn((k, n), generator=g, device=dev, dtype=torch.float32)
            return (w * (init_scale / math.sqrt(k))).to(torch.bfloat16)

        def norm_w(n):
            return (1.0 + 0.05 * torch.randn((n,), generator=g, device=dev)).to(torch.bfloat16)

        self.layers = []
        for _ in range(n_layers):
            self.layers.append(dict(w_in=norm_w(hidden), w_qkv=mat(hidden, (hq + 2 * hkv) * d),
                                    w_o=mat(hq * d, hidden), w_post=norm_w(hidden),
                                    w_gu=mat(hidden, 2 * inter), w_down=mat(inter, hidden)))

    def weight_bytes(self):
        return sum(t.numel() * 2 for lw in self.layers for t in lw.values())

    def flops_per_token(self):
        """GEMM FLOPs per token per step (2 * weights), all layers."""
        per = (self.hidden * (self.hq + 2 * self.hkv) * self.d + self.hq * self.d * self.hidden
               + self.hidden * 2 * self.inter + self.inter * self.hidden)
        return 2.0 * per * self.n_layers

    def buffers(self, n, device="cuda"):
        z = lambda *s: torch.empty(s, dtype=torch.bfloat16, device=device)
        return dict(h=z(n, self.hidden), qkv=z(n, (self.hq + 2 * self.hkv) * self.d),
                    q=z(n, self.hq, self.d), att=z(n, self.hq, self.d), o=z(n, self.hidden),
                    x2=z(n, self.hidden), gu=z(n, 2 * self.inter), a=z(n, self.inter),
                    dn=z(n, self.hidden), xa=z(n, self.hidden), xb=z(n, self.hidden))

    def step(self, x, batch, k_caches, v_caches, pos_base, buf, first_mode=APPEND_ADVANCE,
             stream=None):
        """One decode token for every branch of `batch` through all layers.  x: residual stream
        [n, hidden] bf16 (the token embeddings); k/v_caches: per layer; pos_base: device int32.
        Layer 0 appends with `first_mode` (ADVANCE: the step's new slot), the others REWRITE the
        same slot.  Returns the output residual stream (a buffer of `buf`)."""
        res, dn = x, None
        for l, lw in enumerate(self.layers):
            if dn is None:
                rmsnorm(res, lw["w_in"], out=buf["h"], eps=self.eps, stream=stream)
            else:
                nxt = buf["xa"] if res is not buf["xa"] else buf["xb"]
                rmsnorm(res, lw["w_in"], out=buf["h"], b=dn, residual_out=nxt, eps=self.eps, stream=stream)
                res = nxt
            torch.matmul(buf["h"], lw["w_qkv"], out=buf["qkv"])
            batch.rope_append(buf["qkv"], buf["q"], k_caches[l], v_caches[l], pos_base, self.theta,
                              first_mode if l == 0 else APPEND_REWRITE, stream)
            batch.attend(buf["q"], buf["att"], k_caches[l], v_caches[l], stream=stream)
            torch.matmul(buf["att"].view(-1, self.hq * self.d), lw["w_o"], out=buf["o"])
            rmsnorm(res, lw["w_post"], out=buf["h"], b=buf["o"], residual_out=buf["x2"], eps=self.eps,
                    stream=stream)
            res = buf["x2"]
            torch.matmul(buf["h"], lw["w_gu"], out=buf["gu"])
            silu_mul(buf["gu"], buf["a"], stream=stream)
            torch.matmul(buf["a"], lw["w_down"], out=buf["dn"])
            dn = buf["dn"]
        out = buf["xa"] if res is not buf["xa"] else buf["xb"]
        rmsnorm(res, self.layers[-1]["w_in"], b=dn, residual_out=out, eps=self.eps, stream=stream)
        return out
