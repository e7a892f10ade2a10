"""Hardware-in-the-loop engine: the reference's virtual clock advanced by measured GPU time.

ragsim prices every admitted prefill with ``interpolate(profile, alpha, beta)``
(simulator.py:506) and schedules its first chunk from it (:507-514).
``TimedEngine`` keeps every decision of the reference (it subclasses
``TieredEngine``, which subclasses ragsim's ``SimulationEngine``). The prefill
of each admitted generation is RUN on the GPU: the random-init model's GEMMs,
our K/V write and prefix-prefill kernels, on the generation's real block table
in the device pool. Its CUDA-event time replaces the interpolated cost before
the first chunk is scheduled. The transfer part stays the reference's PCIe
model, fed with the measured GB/s. PGDSF's cost samples (tree.py:240) keep
using the profile. SURVEY.md §8f.2.

Mechanics: ``SimulationEngine._admit`` ends with exactly one ``self._schedule``
call. TimedEngine shadows ``_schedule`` for the duration of ``super()._admit``,
asks the executor for the measured prefill time, recomputes the chunking with the
reference's formula (simulator.py:507-509) and then schedules.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import kernels
from .cache import TieredEngine
from .model import DIMS, PrefillModel, init_weights, suffix_slots
from .synth import _hash32_np


class TimedEngine(TieredEngine):
    """``executor.on_admit(engine, gen, blocks, valid)`` must set ``executor.last_ms``."""

    def __init__(self, *args, executor, **kwargs) -> None:
        super().__init__(*args, executor=executor, **kwargs)
        self.measured: list[tuple[int, int, int, float, float]] = []  # (req, alpha, beta, profile ms, measured ms)
        # (req, modeled transfer ms, charged transfer ms, charged prefill ms) per admission
        self.critical: list[tuple[int, float, float, float]] = []

    def _admit(self, gen) -> None:
        held = []
        self._schedule = lambda *a: held.append(a)  # instance attribute shadows the method
        try:
            super()._admit(gen)
        finally:
            del self._schedule
        if len(held) != 1:
            raise RuntimeError(f"_admit scheduled {len(held)} events; the hook expects 1")
        _, kind, rid, payload = held[0]
        modeled = gen.prefill_ms
        modeled_transfer = gen.transfer_ms
        gen.prefill_ms = float(self.executor.last_ms)
        if getattr(self.executor, "last_transfer_ms", None) is not None:
            # the swap-in was executed and is inside the measured time (serial or
            # layer-pipelined); only its exposed part remains on the critical path
            gen.transfer_ms = float(self.executor.last_transfer_ms)
        total = gen.transfer_ms + gen.prefill_ms
        chunks = max(1, math.ceil(total / self.config.prefill_chunk_ms)) if total > 0 else 1
        gen.chunk_ms = total / chunks
        gen.chunks_left = chunks
        self.measured.append((gen.request.id, gen.alpha, gen.beta, modeled, gen.prefill_ms))
        self.critical.append((gen.request.id, modeled_transfer, gen.transfer_ms, gen.prefill_ms))
        self._schedule(self._now + gen.chunk_ms, kind, rid, payload)


def run_timed(config, trace, sizes, *, pool, executor, stage_provider=None):
    engine = TimedEngine(config, trace, sizes, stage_provider=stage_provider, pool=pool,
                         executor=executor)
    return engine.run(), engine


def doc_tokens(doc: int, n: int, vocab: int, seed: int = 0) -> np.ndarray:
    """Token ids of document ``doc`` (a counter hash of (seed, doc, position)), so every
    prefix path recomputes a document from the same tokens."""
    t = np.arange(n, dtype=np.int64)
    x = (np.int64(doc) * 0x9E3779B1 + t * 0x85EBCA77 + (seed & 0xFFFF) * 0xC2B2AE3D) & 0xFFFFFFFF
    return (_hash32_np(x) % vocab).astype(np.int64)


class ModelExecutor:
    """Runs an admitted generation's prefill on the device pool and times it.

    The suffix = the miss documents then the prompt, in the generation's segment order
    (``GenContext``), written into its reserved suffix pages; cached prefix pages (matched
    nodes, swapped in by the pool if they came from the host tier) are read through the
    block table.  Copies and compute are ordered with the pool's stream fences.

    ``swap_in`` chooses how a generation's host-tier hits (load_to_gpu, tree.py:296-318)
    reach the prefill:
      * ``"modeled"``: the pool copies them before the timed region and the reference's
        ``transfer_time`` (cost_model.py:120-124, measured GB/s) is charged, serially,
        as ragsim does (simulator.py:505-507);
      * ``"serial"``: the H2D copies run inside the timed region, then the prefill;
      * ``"layered"``: the copies are issued per group of ``layers_per_group`` layers and
        layer l's attention waits only for its group, so the transfer
        overlaps the earlier layers' compute.
    In the two measured modes the swap-in time is part of ``last_ms`` and
    ``last_transfer_ms`` is 0.  Swap-outs issued by the admission are drained before the
    timed region in every mode (the reference keeps them off the critical path)."""

    def __init__(self, pool, shape: str, *, seed: int = 0, device="cuda", swap_in: str = "modeled",
                 layers_per_group: int = 4) -> None:
        if swap_in not in ("modeled", "serial", "layered"):
            raise ValueError(f"swap_in must be modeled, serial or layered, not {swap_in!r}")
        self.swap_in = swap_in
        self.layers_per_group = layers_per_group
        self.last_transfer_ms = None
        self.dims = DIMS[shape]
        self.pool = pool
        self.w = init_weights(self.dims, seed=seed, device=device)
        self.model = PrefillModel(self.dims, self.w, block_tokens=pool.block_tokens,
                                  num_pool_blocks=pool.num_gpu_blocks, pool_base=pool.gpu_base)
        self.stream = torch.cuda.current_stream()
        self.device = device
        self.seed = seed
        self.last_ms = 0.0

    def on_admit(self, engine, gen, blocks, valid) -> None:
        ctx = gen.pool_ctx
        bt = self.pool.block_tokens
        alpha, beta = gen.alpha, gen.beta
        parts = [doc_tokens(d, engine.sizes[d], self.dims.vocab, self.seed)
                 for d in ctx.seg_docs if d is not None]
        parts.append(doc_tokens(-1 - gen.request.id, gen.request.prompt_tokens, self.dims.vocab,
                                self.seed))
        tok = torch.from_numpy(np.concatenate(parts)).to(self.device)
        n_prefix = sum(-(-n.size // bt) for n in gen.matched_nodes)
        slots, pos = suffix_slots(blocks, valid, n_prefix, bt, alpha)
        plan = kernels.AttnPlan([(beta, alpha, blocks, valid)], block_tokens=bt,
                                n_q_heads=self.dims.shape.n_q_heads,
                                n_kv_heads=self.dims.shape.n_kv_heads, device=self.device)
        idx = kernels._upload(np.asarray(pos + slots, dtype=np.int32), self.device)
        last = torch.tensor([beta - 1], device=self.device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        fence = None
        if self.swap_in == "modeled":
            self.pool.fence_into(self.stream)  # swap-ins landed before the prefill reads them
            e0.record(self.stream)
        else:
            self.pool.drain()  # this admission's swap-outs: off the critical path
            e0.record(self.stream)
            self.pool.wait_for(self.stream)  # copies start inside the timed region
            if self.swap_in == "layered":
                self.pool.flush_layered(self.layers_per_group)
                fence = lambda layer: self.pool.fence_layer(layer, self.stream)  # noqa: E731
            else:
                self.pool.fence_into(self.stream)
        self.model.prefill(tok, idx[:beta], idx[beta:], plan, last, layer_fence=fence)
        e1.record(self.stream)
        self.pool.wait_for(self.stream)  # later swap-outs read the finished pages
        e1.synchronize()
        self.last_ms = e0.elapsed_time(e1)
        self.last_transfer_ms = None if self.swap_in == "modeled" else 0.0


class ProfileExecutor:
    """Returns the engine profile's own interpolation: TimedEngine then reproduces
    ragsim.run exactly (the interception check)."""

    def __init__(self) -> None:
        from ragsim.cost_model import interpolate

        self.interpolate = interpolate
        self.last_ms = 0.0

    def on_admit(self, engine, gen, blocks, valid) -> None:
        self.last_ms = self.interpolate(engine.profile, gen.alpha, gen.beta)
