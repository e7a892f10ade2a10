"""Measured B200 prefill profile T(alpha, beta) for ragsim's cost model.

ragsim prices a prefill with a profiled grid ``T(alpha cached, beta new)``
(cost_model.py:40-67, bilinear ``interpolate`` :106-117) read from
``RunConfig.profile_path`` (config.py:43,59-61) and consumed both for request
latency (simulator.py:506) and for PGDSF's per-token cost samples
(tree.py:240).  Its default grid is synthetic (cost_model.py:127-147).

``measure_profile`` times the real thing on the GPU: a random-init model of
the requested shape (cuBLAS GEMMs + our RoPE/KV-write + prefix-prefill
attention kernels) prefilling beta suffix tokens on top of alpha cached
tokens held in pool pages, CUDA-event timed, median of ``reps``.  The result
is a ragsim ``CostProfile`` (and CSV via ``save_profile_csv``), so the
reference's engine — decisions unchanged — runs on B200 costs.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels
from ._ragsim import import_ragsim
from .model import DIMS, PrefillModel, init_weights

import_ragsim()
from ragsim.cost_model import DEFAULT_GRID, CostProfile  # noqa: E402


# ragsim's default knots (cost_model.py:29) plus small-beta knots: a cached-prefix
# request computes only its prompt (32 tokens), which the default grid would
# interpolate toward T(alpha, 0) = 0; beta = 1 is one decode step of one request
BETA_GRID = (0, 1, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096)


def _grouped_ok() -> bool:
    from . import model as _model

    return bool(_model._GROUPED_MM)


def decode_ms_per_token(profile, context_tokens: int) -> float:
    """One decode step of one request = a one-token prefill over its cached context:
    the model forward with the same GEMMs and the prefix-prefill kernel as the paged
    decode attention.  Replaces ragsim's constant decode_ms_per_token (config.py:52,
    consumed at simulator.py:419-436)."""
    from ragsim.cost_model import interpolate

    return float(interpolate(profile, context_tokens, 1))


def measure_profile(shape: str = "mistral-7b", alpha_grid=DEFAULT_GRID, beta_grid=BETA_GRID,
                    *, block_tokens: int = 64, reps: int = 5, seed: int = 0, device="cuda",
                    cuda_graph: bool = True) -> tuple[CostProfile, dict]:
    dims = DIMS[shape]
    s = dims.shape
    w = init_weights(dims, seed=seed, device=device)
    max_tok = max(alpha_grid) + max(beta_grid) + block_tokens
    nb = -(-max_tok // block_tokens) + 4
    pool = torch.zeros((nb, s.n_layers, 2, s.n_kv_heads, block_tokens, s.head_dim),
                       dtype=torch.bfloat16, device=device)
    model = PrefillModel(dims, w, block_tokens=block_tokens, num_pool_blocks=nb,
                         pool_base=pool.data_ptr())
    g = torch.Generator(device="cpu").manual_seed(seed)
    times = []
    for a in alpha_grid:
        row = []
        for b in beta_grid:
            if b == 0:
                row.append(0.0)  # nothing to compute (ragsim never asks: prompt >= 1 token)
                continue
            n_a = -(-a // block_tokens)
            n_b = -(-b // block_tokens)
            blocks = list(range(n_a + n_b))
            valid = ([block_tokens] * (n_a - 1) + [a - (n_a - 1) * block_tokens] if a else []) + \
                    [block_tokens] * (n_b - 1) + [b - (n_b - 1) * block_tokens]
            plan = kernels.AttnPlan([(b, a, blocks, valid)], block_tokens=block_tokens,
                                    n_q_heads=s.n_q_heads, n_kv_heads=s.n_kv_heads, device=device)
            slots, pos = [], []
            t = 0
            for blk, v in zip(blocks[n_a:], valid[n_a:]):
                for o in range(v):
                    slots.append(blk * block_tokens + o)
                    pos.append(a + t)
                    t += 1
            tok = torch.randint(0, dims.vocab, (b,), generator=g).to(device)
            pos_t = torch.tensor(pos, dtype=torch.int32, device=device)
            slot_t = torch.tensor(slots, dtype=torch.int32, device=device)
            last = torch.tensor([b - 1], device=device)
            fn = lambda: model.prefill(tok, pos_t, slot_t, plan, last)
            fn()
            fn()
            # a MoE model without the grouped GEMM syncs on its expert offsets: eager
            from . import model as _model
            if cuda_graph and (not dims.n_experts or _model._GROUPED_MM):
                # one graph per (alpha, beta): every layer's GEMMs and rcb kernels
                # replay without per-launch host overhead
                graph = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    fn()
                torch.cuda.current_stream().wait_stream(side)
                with torch.cuda.graph(graph):
                    fn()
                fn = graph.replay
                fn()
            ts = []
            for _ in range(reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            row.append(float(np.median(ts)))
        # ragsim requires T non-decreasing in beta (cost_model.py:64-66)
        row = [float(x) for x in np.maximum.accumulate(row)]
        times.append(tuple(row))
    del w, pool, model
    torch.cuda.empty_cache()
    prof = CostProfile(tuple(alpha_grid), tuple(beta_grid), tuple(times))
    info = {"shape": shape, "block_tokens": block_tokens, "reps": reps,
            "weights": "random-init bf16 (seeded)",
            "timing": "CUDA events, median" + (", CUDA-graph replay" if cuda_graph and (
                not dims.n_experts or _grouped_ok()) else ", eager")}
    return prof, info
