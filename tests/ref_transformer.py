"""Plain PyTorch fp32 reference of the device transformer forward (tests only).

It mirrors the kernels' definition: bf16 weights, fp32 accumulation, bf16 rounding at the same
points (normed activations, qkv, roped q/k, attention output, SiLU*up), fp32 residual stream and
logits.  Weights are read back from the device model through dbl_transformer_get_weight.

fold=True (default) mirrors the kernel's folded RMSNorm exactly: the norm weights of this random-init
family are 1, so RMSNorm(x) @ W^T == rstd(x) * (x @ W^T); the kernel feeds bf16(x) (the residual's
bf16 copy) to the tensor cores and scales the fp32 GEMM output column by rstd (fwd.cuh), where an
HF-style reference rounds bf16(x * rstd).  fold=False is that HF-style rounding point; the two differ
by bf16 re-rounding noise only (~1 % of max|logit| on 2-layer Qwen3-14B shapes).
"""
from __future__ import annotations

import math

import torch


def _bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


class RefTransformer:
    def __init__(self, model, preset_cfg, device: str = "cpu", fold: bool = True):
        c = preset_cfg
        self.c = c
        self.dev = device
        self.fold = fold
        L, h, f, nh, nkv, hd, V = (c.n_layers, c.hidden, c.ffn, c.n_heads, c.n_kv_heads, c.head_dim, c.vocab)
        t = lambda a: torch.from_numpy(a.copy()).to(device)  # noqa: E731
        self.embed = t(model.weight("embed", -1, (V, h)))
        self.lm = t(model.weight("lm_head", -1, (V, h)))
        self.final_norm = t(model.weight("final_norm", -1, (h,)))
        self.layers = []
        for l in range(L):
            d = {
                "attn_norm": t(model.weight("attn_norm", l, (h,))),
                "mlp_norm": t(model.weight("mlp_norm", l, (h,))),
                "q": t(model.weight("q_proj", l, (nh * hd, h))),
                "k": t(model.weight("k_proj", l, (nkv * hd, h))),
                "v": t(model.weight("v_proj", l, (nkv * hd, h))),
                "o": t(model.weight("o_proj", l, (h, nh * hd))),
                "g": t(model.weight("gate_proj", l, (f, h))),
                "u": t(model.weight("up_proj", l, (f, h))),
                "d": t(model.weight("down_proj", l, (h, f))),
            }
            if c.qk_norm:
                d["qn"] = t(model.weight("q_norm", l, (hd,)))
                d["kn"] = t(model.weight("k_norm", l, (hd,)))
            self.layers.append(d)

    def _norm_mm(self, x, w, W, eps):
        """fp32 RMSNorm(x; w) @ W^T at the kernel's (fold) or the HF-style rounding point."""
        if self.fold:
            assert bool((w == 1).all()), "fold mode needs unit norm weights (the kernel folds them)"
            return (_bf(x) @ W.T) * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)
        return self._rms(x, w, eps) @ W.T

    def _rms(self, x, w, eps):
        r = torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)
        return _bf(x * r * w)

    def _rope(self, x, pos):  # x [T, H, hd]
        hd = x.shape[-1]
        half = hd // 2
        # the device RoPE table is computed in fp64 and rounded to fp32 (transformer.cu make_cache)
        i = torch.arange(half, dtype=torch.float64, device=x.device)
        inv = torch.pow(torch.tensor(self.c.rope_theta, dtype=torch.float64, device=x.device), -2.0 * i / hd)
        ang = pos[:, None].to(torch.float64) * inv[None, :]
        cs, sn = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]
        a, b = x[..., :half], x[..., half:]
        return _bf(torch.cat([a * cs - b * sn, b * cs + a * sn], dim=-1))

    @torch.no_grad()
    def logits(self, tokens, first_row: int = 0) -> torch.Tensor:
        """fp32 logits for positions [first_row, len(tokens)) of `tokens` (full causal recompute)."""
        c = self.c
        T = len(tokens)
        nh, nkv, hd, eps = c.n_heads, c.n_kv_heads, c.head_dim, c.rms_eps
        dev = self.dev
        x = self.embed[torch.tensor(tokens, device=dev)].clone()
        pos = torch.arange(T, device=dev)
        mask = torch.tril(torch.ones(T, T, dtype=torch.bool, device=dev))
        for d in self.layers:
            an = d["attn_norm"]
            q = _bf(self._norm_mm(x, an, d["q"], eps)).view(T, nh, hd)
            k = _bf(self._norm_mm(x, an, d["k"], eps)).view(T, nkv, hd)
            v = _bf(self._norm_mm(x, an, d["v"], eps)).view(T, nkv, hd)
            if c.qk_norm:
                q = self._rms(q, d["qn"], eps)
                k = self._rms(k, d["kn"], eps)
            q, k = self._rope(q, pos), self._rope(k, pos)
            g = nh // nkv
            k = k.repeat_interleave(g, dim=1)
            v = v.repeat_interleave(g, dim=1)
            s = torch.einsum("thd,shd->hts", q, k) / math.sqrt(hd)
            s = s.masked_fill(~mask[None], float("-inf"))
            p = torch.softmax(s, dim=-1)
            a = _bf(torch.einsum("hts,shd->thd", p, v)).reshape(T, nh * hd)
            x = x + a @ d["o"].T
            mn = d["mlp_norm"]
            gg, uu = self._norm_mm(x, mn, d["g"], eps), self._norm_mm(x, mn, d["u"], eps)
            act = _bf(gg / (1 + torch.exp(-gg)) * uu)
            x = x + act @ d["d"].T
        return self._norm_mm(x[first_row:], self.final_norm, self.lm, eps).cpu()
