"""Random-init LLaMA/Mistral-shape decoder for prefix-cached prefill.

The dense projections and MLP are plain library GEMMs (torch.matmul ->
cuBLAS); every attention-side op is ours: RoPE + paged KV write
(rcb_kv_write_rope) and prefix-aware attention over the block table
(rcb_prefix_prefill).  A request's cached documents are never recomputed:
their K/V pages are read from the pool, and only the suffix tokens (miss
docs + prompt) flow through the layers (the 11.5x
cached-prefix prefill; ragsim models it as T(alpha, beta),
cost_model.py:106-117).

Used for (a) logits parity of cached-prefix prefill against an fp32 oracle
(tests/test_gpu_model.py) and (b) measuring the B200 T(alpha, beta) grid that
replaces ragsim's synthetic profile (profile.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import kernels
from .workloads import SHAPES, ModelShape


@dataclass(frozen=True)
class ModelDims:
    shape: ModelShape
    d_model: int
    ffn: int
    vocab: int
    norm_eps: float = 1e-5
    n_experts: int = 0  # > 0: sparse MoE FFN (Mixtral), top_k experts per token
    top_k: int = 2


DIMS = {
    "tiny": ModelDims(SHAPES["tiny"], 256, 688, 1024),
    "mistral-7b": ModelDims(SHAPES["mistral-7b"], 4096, 14336, 32000),
    "llama2-7b": ModelDims(SHAPES["llama2-7b"], 4096, 11008, 32000),
    "llama2-13b": ModelDims(SHAPES["llama2-13b"], 5120, 13824, 32000),
    # configs[4]: Mixtral-8x7B (32 layers, GQA 32/8, 8 experts of FFN 14336, top-2;
    # ~93 GB of bf16 weights, one B200)
    "mixtral-8x7b": ModelDims(SHAPES["mixtral-8x7b"], 4096, 14336, 32000, n_experts=8, top_k=2),
}


def init_weights(dims: ModelDims, seed: int = 0, device="cuda", dtype=torch.bfloat16):
    """Seeded random weights (fan-in scaled so activations stay O(1))."""
    s = dims.shape
    gen_dev = "cpu" if str(device) == "cpu" or dims.d_model <= 1024 else device
    g = torch.Generator(device=gen_dev)  # big models: generate on the device
    g.manual_seed(seed)

    def w(rows, cols, scale=1.0):
        t = torch.randn((rows, cols), generator=g, device=gen_dev) * (scale / rows ** 0.5)
        return t.to(device=device, dtype=dtype)

    def experts(rows, cols):  # [E, rows, cols], one matrix per expert
        return torch.stack([w(rows, cols) for _ in range(dims.n_experts)])

    qkv = (s.n_q_heads + 2 * s.n_kv_heads) * s.head_dim
    layers = []
    for _ in range(s.n_layers):
        lw = {
            "ln1": (1.0 + 0.1 * torch.randn(dims.d_model, generator=g, device=gen_dev)).to(device, dtype),
            "wqkv": w(dims.d_model, qkv),
            "wo": w(s.n_q_heads * s.head_dim, dims.d_model),
            "ln2": (1.0 + 0.1 * torch.randn(dims.d_model, generator=g, device=gen_dev)).to(device, dtype),
        }
        if dims.n_experts:
            lw["router"] = w(dims.d_model, dims.n_experts)
            lw["wgu"] = experts(dims.d_model, 2 * dims.ffn)
            lw["wdown"] = experts(dims.ffn, dims.d_model)
        else:
            lw["wgu"] = w(dims.d_model, 2 * dims.ffn)
            lw["wdown"] = w(dims.ffn, dims.d_model)
        layers.append(lw)
    return {
        "emb": (torch.randn((dims.vocab, dims.d_model), generator=g, device=gen_dev)).to(device, dtype),
        "layers": layers,
        "norm": torch.ones(dims.d_model).to(device, dtype),
        "lm_head": w(dims.d_model, dims.vocab, 0.5),
    }


class PrefillModel:
    def __init__(self, dims: ModelDims, weights, *, block_tokens: int, num_pool_blocks: int,
                 pool_base: int) -> None:
        self.dims = dims
        self.w = weights
        self.bt = block_tokens
        self.nb = num_pool_blocks
        self.base = pool_base
        self.rope = kernels.rope_table(1 << 14, dims.shape.head_dim, dims.shape.rope_theta,
                                       device=weights["emb"].device)

    def prefill(self, tokens: torch.Tensor, positions: torch.Tensor, slots: torch.Tensor,
                plan: "kernels.AttnPlan", last_rows: torch.Tensor, stream=None,
                layer_fence=None) -> torch.Tensor:
        """tokens/positions/slots: [T] suffix tokens of all requests (packed in plan
        order); returns fp32 logits [len(last_rows), vocab] of the rows last_rows.
        ``layer_fence(layer)`` (optional) runs before a layer's attention reads the
        cached pages: the layer-pipelined swap-in waits there for that layer's copies
        only (BlockPool.fence_layer), the suffix K/V write never touches them."""
        d = self.dims
        s = d.shape
        T = tokens.shape[0]
        x = self.w["emb"][tokens].float()  # residual stream kept in fp32; bf16 into GEMMs
        bf = self.w["emb"].dtype
        attn = torch.empty((T, s.n_q_heads, s.head_dim), dtype=bf, device=x.device)
        qw = s.n_q_heads * s.head_dim
        kw = s.n_kv_heads * s.head_dim
        layers = self.w["layers"]
        # residual add + RMSNorm and SiLU * up run as one kernel each (rcb_rmsnorm_residual,
        # rcb_silu_mul); the projections are library GEMMs
        h = kernels.rmsnorm_residual(x, None, layers[0]["ln1"], d.norm_eps, stream=stream)
        for layer, lw in enumerate(layers):
            qkv = h @ lw["wqkv"]
            # K/V rotated into the pool; Q's RoPE runs inside the attention kernel
            kernels.kv_write_rope(None, qkv[:, qw:qw + kw], qkv[:, qw + kw:], None, positions,
                                  slots, self.base, block_tokens=self.bt, n_layers=s.n_layers,
                                  n_kv_heads=s.n_kv_heads, head_dim=s.head_dim, layer=layer,
                                  rope_theta=s.rope_theta, n_q_heads=s.n_q_heads, stream=stream)
            if layer_fence is not None:
                layer_fence(layer)
            kernels.prefix_prefill(qkv[:, :qw], attn, plan, self.base, self.nb,
                                   block_tokens=self.bt, n_layers=s.n_layers,
                                   n_kv_heads=s.n_kv_heads, head_dim=s.head_dim, layer=layer,
                                   rope=self.rope, n_q_heads=s.n_q_heads, stream=stream)
            h = kernels.rmsnorm_residual(x, attn.view(T, qw) @ lw["wo"], lw["ln2"], d.norm_eps,
                                         stream=stream)
            if d.n_experts:
                mlp = moe_ffn(h, lw, d, stream=stream)
            else:
                mlp = kernels.silu_mul(h @ lw["wgu"], stream=stream) @ lw["wdown"]
            nxt = layers[layer + 1]["ln1"] if layer + 1 < len(layers) else self.w["norm"]
            h = kernels.rmsnorm_residual(x, mlp, nxt, d.norm_eps, stream=stream)
        # logits leave the GEMM in fp32 (cuBLAS accumulates in fp32 either way): a bf16
        # output would add a rounding of up to |logit| * 2^-9 on top of the activations'
        return _mm_f32(h[last_rows], self.w["lm_head"])


def _mm_f32(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """bf16 GEMM with an fp32 output (cuBLAS accumulates in fp32; no bf16 output rounding)."""
    if a.is_cuda:
        return torch.mm(a, b, out_dtype=torch.float32)
    return a.float() @ b.float()


_GROUPED_MM = None  # torch._grouped_mm usable on this device (probed on first use)


def _grouped(x: torch.Tensor, w3: torch.Tensor, offs: torch.Tensor) -> torch.Tensor:
    """rows [offs[e-1], offs[e]) of x times w3[e]: one grouped GEMM (no host sync, CUDA-graph
    capturable); a per-expert loop over library GEMMs where the grouped kernel is missing."""
    global _GROUPED_MM
    if _GROUPED_MM is not False:
        try:
            y = torch._grouped_mm(x, w3, offs=offs)
            _GROUPED_MM = True
            return y
        except (RuntimeError, NotImplementedError, AttributeError):
            if _GROUPED_MM:
                raise
            _GROUPED_MM = False
    ends = offs.tolist()
    out = torch.empty((x.shape[0], w3.shape[2]), dtype=x.dtype, device=x.device)
    lo = 0
    for e, hi in enumerate(ends):
        if hi > lo:
            torch.mm(x[lo:hi], w3[e], out=out[lo:hi])
        lo = hi
    return out


def moe_ffn(h: torch.Tensor, lw, dims: ModelDims, stream=None) -> torch.Tensor:
    """Mixtral sparse FFN on bf16 rows h [T, d]: router logits in fp32, top-k experts per
    token, their softmax-renormalised weights; the T*k (token, expert) rows are sorted by
    expert and run through per-expert gate/up and down GEMMs (grouped), then combined
    into bf16 [T, d].  The combine adds the k fp32 contributions to a zero row, which is
    order-independent (two addends), so the result is deterministic."""
    T = h.shape[0]
    k = dims.top_k
    logits = _mm_f32(h, lw["router"])
    top_v, top_i = torch.topk(logits, k, dim=-1)
    wts = torch.softmax(top_v, dim=-1).reshape(-1)
    flat = top_i.reshape(-1)
    order = torch.argsort(flat, stable=True)
    tok = order // k
    counts = torch.zeros(dims.n_experts, dtype=torch.int64, device=h.device)
    counts.scatter_add_(0, flat, torch.ones_like(flat))  # (bincount would sync on its max)
    offs = torch.cumsum(counts, 0).to(torch.int32)
    gu = _grouped(h[tok], lw["wgu"], offs)
    y = _grouped(kernels.silu_mul(gu, stream=stream), lw["wdown"], offs)
    out = torch.zeros((T, h.shape[1]), dtype=torch.float32, device=h.device)
    out.index_add_(0, tok, y.float() * wts[order][:, None])
    return out.to(h.dtype)


def suffix_slots(blocks, valid, n_prefix_blocks: int, block_tokens: int, alpha: int):
    """Pool slots and logical positions of a request's suffix tokens."""
    slots, pos = [], []
    t = 0
    for b, v in zip(blocks[n_prefix_blocks:], valid[n_prefix_blocks:]):
        for o in range(v):
            slots.append(b * block_tokens + o)
            pos.append(alpha + t)
            t += 1
    return slots, pos
