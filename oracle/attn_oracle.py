"""ORACLE (test infrastructure only — never imported by the product path).

fp32 CPU restatement of prefix-aware prefill attention over a paged KV pool,
plus RoPE.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
leg may import this module.

Reference anchoring: ragsim has NO attention arithmetic — its prefill is the
latency stand-in T(alpha, beta) (cost_model.py:106-117, used at
simulator.py:506 and tree.py:240).  The semantics restated here are the
paper's: a request's KV is the concatenation of the cached per-node KV along
the knowledge-tree path ("order-dependent KV per path
node") held in non-contiguous blocks, followed by the
uncached suffix; only the suffix tokens are queries, causal on logical
positions.  Parity for KV/attention values is therefore UNPINNED by the
reference and checked against this fp32 restatement within
a stated bf16 tolerance.
"""

from __future__ import annotations

import math

import torch


def rope_inv_freq(head_dim: int, theta: float) -> torch.Tensor:
    return 1.0 / (theta ** (torch.arange(0, head_dim, 2, dtype=torch.float32) / head_dim))


def apply_rope(x: torch.Tensor, positions: torch.Tensor, theta: float) -> torch.Tensor:
    """Rotate-half RoPE (LLaMA convention) in fp32. x: [T, H, d], positions: [T]."""
    d = x.shape[-1]
    inv = rope_inv_freq(d, theta).to(x.device)
    ang = positions.to(x.device, torch.float32)[:, None] * inv[None, :]
    cos, sin = ang.cos()[:, None, :], ang.sin()[:, None, :]
    x = x.to(torch.float32)
    x0, x1 = x[..., : d // 2], x[..., d // 2:]
    return torch.cat([x0 * cos - x1 * sin, x1 * cos + x0 * sin], dim=-1)


def pool_view(pool_bytes: torch.Tensor, n_blocks: int, n_layers: int, n_kv_heads: int,
              block_tokens: int, head_dim: int) -> torch.Tensor:
    """Interpret raw pool bytes as bf16 [NB][L][2][Hkv][B][d] (block-major pages)."""
    return pool_bytes.view(torch.bfloat16).view(n_blocks, n_layers, 2, n_kv_heads, block_tokens,
                                                 head_dim)


def gather_request_kv(pool: torch.Tensor, layer: int, blocks, valid):
    """K, V [Hkv, S, d] fp32 of a block table with per-block valid tokens."""
    ks, vs = [], []
    for b, v in zip(blocks, valid):
        ks.append(pool[int(b), layer, 0, :, : int(v), :].to(torch.float32))
        vs.append(pool[int(b), layer, 1, :, : int(v), :].to(torch.float32))
    return torch.cat(ks, dim=1), torch.cat(vs, dim=1)


def prefix_prefill(q: torch.Tensor, pool: torch.Tensor, requests, layer: int,
                   softmax_scale: float | None = None) -> torch.Tensor:
    """q: [T_total, Hq, d] (post-RoPE); requests: [(q_len, q_pos0, blocks, valid)].

    Returns fp32 [T_total, Hq, d] on q's device (a CUDA q and pool run this fp32
    restatement on the GPU: the plain-PyTorch fp32 reference at sizes the host cannot
    finish in seconds; TF32 must be off)."""
    t_total, hq, d = q.shape
    hkv = pool.shape[3]
    g = hq // hkv
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(d)
    dev = q.device
    out = torch.zeros((t_total, hq, d), dtype=torch.float32, device=dev)
    start = 0
    for q_len, q_pos0, blocks, valid in requests:
        k, v = gather_request_kv(pool, layer, blocks, valid)  # [Hkv, S, d]
        s_len = k.shape[1]
        assert s_len == q_pos0 + q_len, "block table must cover prefix + suffix"
        kq = k.repeat_interleave(g, dim=0)  # [Hq, S, d]
        vq = v.repeat_interleave(g, dim=0)
        qr = q[start:start + q_len].to(torch.float32).permute(1, 0, 2)  # [Hq, t, d]
        scores = torch.matmul(qr, kq.transpose(1, 2)) * scale  # [Hq, t, S]
        qpos = q_pos0 + torch.arange(q_len, device=dev)
        kpos = torch.arange(s_len, device=dev)
        mask = kpos[None, :] > qpos[:, None]
        scores = scores.masked_fill(mask[None], float("-inf"))
        p = torch.softmax(scores, dim=-1)
        out[start:start + q_len] = torch.matmul(p, vq).permute(1, 0, 2)
        start += q_len
    return out
