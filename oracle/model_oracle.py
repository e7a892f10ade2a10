"""ORACLE (test infrastructure only — never imported by the product path).

fp32 CPU forward of the LLaMA-style decoder of paper_2404_12457_b200.model
over the FULL token sequence (no KV cache, no paging).  A cached-prefix
prefill on the GPU — prefix KV read from knowledge-tree node pages, only the
suffix computed — must reproduce these logits within the north star's stated
bf16 tolerance (max |logit error| <= 1e-2).  The reference has no model
(its prefill is the latency stand-in cost_model.py:106-117), so this parity
is UNPINNED by the reference and anchored on the paper's semantics: cached
KV is exactly the KV the full sequence would produce.
"""

from __future__ import annotations

import math

import torch

from .attn_oracle import apply_rope


def _rms(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _moe(h, lw, dims, f):
    """Mixtral sparse FFN (the published routing: softmax over the top-k router logits,
    weighted sum of those experts' SwiGLU outputs), fp32, dense per-expert loop."""
    logits = h @ f(lw["router"])
    top_v, top_i = torch.topk(logits, dims.top_k, dim=-1)
    wts = torch.softmax(top_v, dim=-1)
    out = torch.zeros_like(h)
    for e in range(dims.n_experts):
        sel = (top_i == e)
        rows = sel.any(-1).nonzero().reshape(-1)
        if rows.numel() == 0:
            continue
        gu = h[rows] @ f(lw["wgu"][e])
        y = (torch.nn.functional.silu(gu[:, : dims.ffn]) * gu[:, dims.ffn:]) @ f(lw["wdown"][e])
        out[rows] += y * (wts[rows] * sel[rows]).sum(-1, keepdim=True)
    return out


def forward_full(weights, dims, tokens: torch.Tensor, device="cpu",
                 last_only: bool = False) -> torch.Tensor:
    """weights: the model's dict (any dtype/device); returns fp32 logits [S, vocab]
    ([1, vocab] of the last token with last_only).  device="cuda" runs the same fp32
    arithmetic on the GPU (TF32 off) for full-size geometries."""
    s = dims.shape
    f = lambda t: t.detach().to(device, torch.float32)
    S = tokens.shape[0]
    x = f(weights["emb"])[tokens.to(device)]
    pos = torch.arange(S, device=device)
    qw = s.n_q_heads * s.head_dim
    kw = s.n_kv_heads * s.head_dim
    g = s.n_q_heads // s.n_kv_heads
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=device), 1)
    for lw in weights["layers"]:
        h = _rms(x, f(lw["ln1"]), dims.norm_eps)
        qkv = h @ f(lw["wqkv"])
        q = apply_rope(qkv[:, :qw].view(S, s.n_q_heads, s.head_dim), pos, s.rope_theta)
        k = apply_rope(qkv[:, qw:qw + kw].view(S, s.n_kv_heads, s.head_dim), pos, s.rope_theta)
        v = qkv[:, qw + kw:].view(S, s.n_kv_heads, s.head_dim)
        k = k.repeat_interleave(g, 1)
        v = v.repeat_interleave(g, 1)
        sc = torch.einsum("thd,shd->hts", q, k) / math.sqrt(s.head_dim)
        sc = sc.masked_fill(mask[None], float("-inf"))
        o = torch.einsum("hts,shd->thd", torch.softmax(sc, -1), v).reshape(S, qw)
        x = x + o @ f(lw["wo"])
        h = _rms(x, f(lw["ln2"]), dims.norm_eps)
        if getattr(dims, "n_experts", 0):
            x = x + _moe(h, lw, dims, f)
        else:
            gu = h @ f(lw["wgu"])
            x = x + (torch.nn.functional.silu(gu[:, : dims.ffn]) * gu[:, dims.ffn:]) @ f(lw["wdown"])
    if last_only:
        x = x[-1:]
    return _rms(x, f(weights["norm"]), dims.norm_eps) @ f(weights["lm_head"])
