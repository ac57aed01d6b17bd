"""TEST INFRASTRUCTURE: plain-PyTorch restatement of the GPT decoder whose HVP
the product computes (same flat parameter layout as oracle/src/models.cpp
gpt_layout and paper_2505_11564_b200.gpt.param_layout). Used as the
independent float64 reference for the CUDA HVP at shapes the C++ oracle's
tape is too slow for (full GPT-2-small dims), and to cross-check the oracle.
"""
from __future__ import annotations

import math

import torch


def layout(cfg):
    V, S, d, ff = cfg["vocab"], cfg["ctx"], cfg["d"], cfg["ff"]
    out = [("wte", (V, d), 0), ("wpe", (S, d), 0)]
    for l in range(cfg["n_layer"]):
        p = f"h{l}."
        out += [(p + "ln_1.weight", (d,), 1), (p + "ln_1.bias", (d,), 2),
                (p + "attn.c_attn.weight", (d, 3 * d), 0), (p + "attn.c_attn.bias", (3 * d,), 2),
                (p + "attn.c_proj.weight", (d, d), 0), (p + "attn.c_proj.bias", (d,), 2),
                (p + "ln_2.weight", (d,), 1), (p + "ln_2.bias", (d,), 2),
                (p + "mlp.c_fc.weight", (d, ff), 0), (p + "mlp.c_fc.bias", (ff,), 2),
                (p + "mlp.c_proj.weight", (ff, d), 0), (p + "mlp.c_proj.bias", (d,), 2)]
    out += [("ln_f.weight", (d,), 1), ("ln_f.bias", (d,), 2)]
    return out


def unflatten(cfg, flat):
    ps, off = {}, 0
    for name, shape, _ in layout(cfg):
        n = math.prod(shape)
        ps[name] = flat[off:off + n].view(shape)
        off += n
    assert off == flat.numel()
    return ps


def loss_fn(cfg, flat, tok, tgt, B, S, eps=1e-5):
    p = unflatten(cfg, flat)
    d, H = cfg["d"], cfg["n_head"]
    dh = d // H
    tok = tok.view(B, S).long()
    tgt = tgt.view(B, S).long()
    x = p["wte"][tok] + p["wpe"][:S].unsqueeze(0)
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=flat.device), 1)

    def ln(x, g, b):
        mu = x.mean(-1, keepdim=True)
        xc = x - mu
        var = (xc * xc).mean(-1, keepdim=True)
        return xc * torch.rsqrt(var + eps) * g + b

    for l in range(cfg["n_layer"]):
        q = f"h{l}."
        h = ln(x, p[q + "ln_1.weight"], p[q + "ln_1.bias"])
        qkv = h @ p[q + "attn.c_attn.weight"] + p[q + "attn.c_attn.bias"]
        qq, kk, vv = qkv.split(d, dim=-1)
        qq = qq.view(B, S, H, dh).transpose(1, 2)
        kk = kk.view(B, S, H, dh).transpose(1, 2)
        vv = vv.view(B, S, H, dh).transpose(1, 2)
        s = (qq @ kk.transpose(-1, -2)) / math.sqrt(dh)
        s = s.masked_fill(mask, float("-inf"))
        o = torch.softmax(s, -1) @ vv
        o = o.transpose(1, 2).reshape(B, S, d)
        x = x + o @ p[q + "attn.c_proj.weight"] + p[q + "attn.c_proj.bias"]
        h = ln(x, p[q + "ln_2.weight"], p[q + "ln_2.bias"])
        f = h @ p[q + "mlp.c_fc.weight"] + p[q + "mlp.c_fc.bias"]
        f = 0.5 * f * (1.0 + torch.tanh(math.sqrt(2.0 / math.pi) * (f + 0.044715 * f ** 3)))
        x = x + f @ p[q + "mlp.c_proj.weight"] + p[q + "mlp.c_proj.bias"]
    h = ln(x, p["ln_f.weight"], p["ln_f.bias"])
    logits = h @ p["wte"].t()
    return torch.nn.functional.cross_entropy(logits.reshape(B * S, -1), tgt.reshape(-1))


def hvp(cfg, theta, tok, tgt, B, S, v):
    """Pearlmutter double backward (Alg. 1 lines 9-12)."""
    th = theta.detach().clone().requires_grad_(True)
    L = loss_fn(cfg, th, tok, tgt, B, S)
    (g,) = torch.autograd.grad(L, th, create_graph=True)
    (hv,) = torch.autograd.grad((g * v).sum(), th)
    return hv.detach()


def grad(cfg, theta, tok, tgt, B, S):
    th = theta.detach().clone().requires_grad_(True)
    L = loss_fn(cfg, th, tok, tgt, B, S)
    (g,) = torch.autograd.grad(L, th)
    return g.detach(), float(L)
