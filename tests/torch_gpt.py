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


# ---------------------------------------------------------------- Llama-style
# Same decoder as oracle/src/models.cpp build_llama: RMSNorm (pre-norm,
# (mean(x^2) + eps)^-1/2), RoPE rotate-half (theta_i = base^(-2i/dh)), causal
# softmax attention with grouped-query heads (query head h reads kv head
# h // (H / KV)), SwiGLU MLP silu(gate) * up with [gate | up] fused columns,
# untied output head [V][d]; no biases.
def llama_layout(cfg):
    V, d, ff, H = cfg["vocab"], cfg["d"], cfg["ff"], cfg["n_head"]
    KV = cfg.get("n_kv_head") or H
    kvd = KV * (d // H)
    out = [("tok_embeddings", (V, d))]
    for l in range(cfg["n_layer"]):
        p = f"layers.{l}."
        out += [(p + "attention_norm.weight", (d,)), (p + "attention.wqkv", (d, d + 2 * kvd)),
                (p + "attention.wo", (d, d)), (p + "ffn_norm.weight", (d,)),
                (p + "feed_forward.w_gate_up", (d, 2 * ff)), (p + "feed_forward.w_down", (ff, d))]
    out += [("norm.weight", (d,)), ("output", (V, d))]
    return out


def llama_loss_fn(cfg, flat, tok, tgt, B, S, eps=1e-5):
    ps, off = {}, 0
    for name, shape in llama_layout(cfg):
        n = math.prod(shape)
        ps[name] = flat[off:off + n].view(shape)
        off += n
    assert off == flat.numel()
    d, H, ff = cfg["d"], cfg["n_head"], cfg["ff"]
    KV = cfg.get("n_kv_head") or H
    dh, G = d // H, H // KV
    kvd = KV * dh
    base = float(cfg.get("rope_base", 10000.0))
    tok = tok.view(B, S).long()
    tgt = tgt.view(B, S).long()
    x = ps["tok_embeddings"][tok]
    half = dh // 2
    inv = base ** (-2.0 * torch.arange(half, dtype=torch.float64, device=flat.device) / dh)
    ang = torch.arange(S, dtype=torch.float64, device=flat.device)[:, None] * inv[None, :]
    cos = torch.cat([ang.cos(), ang.cos()], -1).to(flat.dtype)
    sin = torch.cat([ang.sin(), ang.sin()], -1).to(flat.dtype)
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=flat.device), 1)

    def rms(x, g):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * g

    def rope(t):  # t: [B, h, S, dh]; (t R)[i] = -t[i + half], (t R)[i + half] = t[i]
        rot = torch.cat([-t[..., half:], t[..., :half]], -1)
        return t * cos + rot * sin

    for l in range(cfg["n_layer"]):
        p = f"layers.{l}."
        h = rms(x, ps[p + "attention_norm.weight"])
        qkv = h @ ps[p + "attention.wqkv"]
        q = qkv[..., :d].reshape(B, S, H, dh).transpose(1, 2)
        k = qkv[..., d:d + kvd].reshape(B, S, KV, dh).transpose(1, 2)
        v = qkv[..., d + kvd:].reshape(B, S, KV, dh).transpose(1, 2)
        q, k = rope(q), rope(k)
        k = k.repeat_interleave(G, dim=1)
        v = v.repeat_interleave(G, dim=1)
        s = (q @ k.transpose(-1, -2)) / math.sqrt(dh)
        s = s.masked_fill(mask, float("-inf"))
        o = (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(B, S, d)
        x = x + o @ ps[p + "attention.wo"]
        h = rms(x, ps[p + "ffn_norm.weight"])
        gu = h @ ps[p + "feed_forward.w_gate_up"]
        gate, up = gu[..., :ff], gu[..., ff:]
        x = x + (gate * torch.sigmoid(gate) * up) @ ps[p + "feed_forward.w_down"]
    h = rms(x, ps["norm.weight"])
    logits = h @ ps["output"].t()
    return torch.nn.functional.cross_entropy(logits.reshape(B * S, -1), tgt.reshape(-1))


def llama_hvp(cfg, theta, tok, tgt, B, S, v):
    th = theta.detach().clone().requires_grad_(True)
    L = llama_loss_fn(cfg, th, tok, tgt, B, S)
    (g,) = torch.autograd.grad(L, th, create_graph=True)
    (hv,) = torch.autograd.grad((g * v).sum(), th)
    return hv.detach()


def any_hvp(cfg, theta, tok, tgt, B, S, v):
    return (llama_hvp if cfg.get("arch", 0) == 1 else hvp)(cfg, theta, tok, tgt, B, S, v)
