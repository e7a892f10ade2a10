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


DIMS = {
    "tiny": ModelDims(SHAPES["tiny"], 256, 688, 1024),
    "mistral-7b": ModelDims(SHAPES["mistral-7b"], 4096, 14336, 32000),
    "llama2-7b": ModelDims(SHAPES["llama2-7b"], 4096, 11008, 32000),
    "llama2-13b": ModelDims(SHAPES["llama2-13b"], 5120, 13824, 32000),
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

    qkv = (s.n_q_heads + 2 * s.n_kv_heads) * s.head_dim
    layers = []
    for _ in range(s.n_layers):
        layers.append({
            "ln1": (1.0 + 0.1 * torch.randn(dims.d_model, generator=g, device=gen_dev)).to(device, dtype),
            "wqkv": w(dims.d_model, qkv),
            "wo": w(s.n_q_heads * s.head_dim, dims.d_model),
            "ln2": (1.0 + 0.1 * torch.randn(dims.d_model, generator=g, device=gen_dev)).to(device, dtype),
            "wgu": w(dims.d_model, 2 * dims.ffn),
            "wdown": w(dims.ffn, dims.d_model),
        })
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
            mlp = kernels.silu_mul(h @ lw["wgu"], stream=stream) @ lw["wdown"]
            nxt = layers[layer + 1]["ln1"] if layer + 1 < len(layers) else self.w["norm"]
            h = kernels.rmsnorm_residual(x, mlp, nxt, d.norm_eps, stream=stream)
        # logits leave the GEMM in fp32 (cuBLAS accumulates in fp32 either way): a bf16
        # output would add a rounding of up to |logit| * 2^-9 on top of the activations'
        return torch.mm(h[last_rows], self.w["lm_head"], out_dtype=torch.float32)


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
