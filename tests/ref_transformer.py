"""Plain PyTorch fp32 reference of the device transformer forward (tests only).

It mirrors the kernels' definition: bf16 weights, fp32 accumulation, bf16 rounding at the same
points (normed activations, qkv, roped q/k, attention output, SiLU*up), fp32 residual stream and
logits.  Weights are read back from the device model through dbl_transformer_get_weight.
"""
from __future__ import annotations

import math

import torch


def _bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


class RefTransformer:
    def __init__(self, model, preset_cfg):
        c = preset_cfg
        self.c = c
        L, h, f, nh, nkv, hd, V = (c.n_layers, c.hidden, c.ffn, c.n_heads, c.n_kv_heads, c.head_dim, c.vocab)
        t = lambda a: torch.from_numpy(a.copy())  # noqa: E731
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

    def _rms(self, x, w, eps):
        r = torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)
        return _bf(x * r * w)

    def _rope(self, x, pos):  # x [T, H, hd]
        hd = x.shape[-1]
        half = hd // 2
        i = torch.arange(half, dtype=torch.float32)
        inv = torch.pow(torch.tensor(self.c.rope_theta, dtype=torch.float32), -2.0 * i / hd)
        ang = pos[:, None].to(torch.float32) * inv[None, :]
        cs, sn = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
        a, b = x[..., :half], x[..., half:]
        return _bf(torch.cat([a * cs - b * sn, b * cs + a * sn], dim=-1))

    @torch.no_grad()
    def logits(self, tokens) -> torch.Tensor:
        """fp32 logits for every position of `tokens` (full causal recompute)."""
        c = self.c
        T = len(tokens)
        nh, nkv, hd, eps = c.n_heads, c.n_kv_heads, c.head_dim, c.rms_eps
        x = self.embed[torch.tensor(tokens)].clone()
        pos = torch.arange(T)
        mask = torch.tril(torch.ones(T, T, dtype=torch.bool))
        for d in self.layers:
            xn = self._rms(x, d["attn_norm"], eps)
            q = _bf(xn @ d["q"].T).view(T, nh, hd)
            k = _bf(xn @ d["k"].T).view(T, nkv, hd)
            v = _bf(xn @ d["v"].T).view(T, nkv, hd)
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
            xn = self._rms(x, d["mlp_norm"], eps)
            gg, uu = xn @ d["g"].T, xn @ d["u"].T
            act = _bf(gg / (1 + torch.exp(-gg)) * uu)
            x = x + act @ d["d"].T
        xn = self._rms(x, self.final_norm, eps)
        return xn @ self.lm.T
