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
        self.skipped_chunks = 0  # chunks of terminated speculations that never ran
        self.planned_chunks = 0  # chunks of every chunked admission (run + skipped)
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
        if getattr(gen, "exec_state", None) is not None:
            # chunked execution (simulator.py:507-510): the executor ran chunk 0 of the
            # reference's chunk count; each later chunk runs at its iteration boundary
            # (_on_prefill_iteration), so a terminated speculation stops launching
            gen.chunk_ms = gen.transfer_ms + gen.prefill_ms
        else:
            total = gen.transfer_ms + gen.prefill_ms
            chunks = max(1, math.ceil(total / self.config.prefill_chunk_ms)) if total > 0 else 1
            gen.chunk_ms = total / chunks
            gen.chunks_left = chunks
        if getattr(gen, "exec_state", None) is not None:
            gen.exec_state["measured_idx"] = len(self.measured)
            self.planned_chunks += gen.chunks_left
        self.measured.append((gen.request.id, gen.alpha, gen.beta, modeled, gen.prefill_ms))
        self.critical.append((gen.request.id, modeled_transfer, gen.transfer_ms, gen.prefill_ms))
        self._schedule(self._now + gen.chunk_ms, kind, rid, payload)

    def _on_prefill_iteration(self, gen) -> None:
        """simulator.py:408-425 with real chunks: at a boundary of a chunked generation that
        goes on (not terminated, chunks left), the next chunk runs on the GPU and its
        measured time is the next iteration's length.  ragsim's bookkeeping (executed_ms +=
        the finished chunk) is kept by pre-compensating executed_ms."""
        st = getattr(gen, "exec_state", None)
        if st is not None and not gen.terminated and gen.chunks_left > 1:
            nxt = float(self.executor.run_chunk(gen, st["n"] - gen.chunks_left + 1))
            gen.executed_ms += gen.chunk_ms - nxt
            gen.chunk_ms = nxt
            gen.prefill_ms += nxt
            self.measured[st["measured_idx"]] = self.measured[st["measured_idx"]][:4] + (
                gen.prefill_ms,)
        elif st is not None and gen.terminated and gen.chunks_left > 1:
            self.skipped_chunks += gen.chunks_left - 1  # never launched
        super()._on_prefill_iteration(gen)


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
                 layers_per_group: int = 4, chunked: bool = False, dims=None,
                 weights=None) -> None:
        if swap_in not in ("modeled", "serial", "layered"):
            raise ValueError(f"swap_in must be modeled, serial or layered, not {swap_in!r}")
        self.swap_in = swap_in
        self.layers_per_group = layers_per_group
        self.last_transfer_ms = None
        self.dims = dims if dims is not None else DIMS[shape]
        # chunked: run the suffix in the reference's chunk count (simulator.py:507-510),
        # one chunk per iteration boundary (TimedEngine._on_prefill_iteration)
        self.chunked = chunked
        self.chunks_run = 0
        self.last_logits = None
        self.pool = pool
        # weights may be shared across executors (one random-init model, many pools)
        self.w = weights if weights is not None else init_weights(self.dims, seed=seed,
                                                                 device=device)
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
        idx = kernels._upload(np.asarray(pos + slots, dtype=np.int32), self.device)
        n = max(1, min(int(gen.chunks_left), beta)) if self.chunked else 1
        st = {"tok": tok, "pos": idx[:beta], "slots": idx[beta:], "blocks": list(blocks),
              "valid": list(valid), "alpha": alpha, "beta": beta, "n": n,
              "cuts": [round(c * beta / n) for c in range(n + 1)]}
        if self.chunked:
            gen.exec_state = st
            gen.chunks_left = n
        self.last_ms = self._run(st, 0, first=True)
        self.last_transfer_ms = None if self.swap_in == "modeled" else 0.0

    def run_chunk(self, gen, c: int) -> float:
        """Chunk c (> 0) of a chunked generation: its tokens over the cached prefix plus the
        earlier chunks' pages (written by their K/V writes)."""
        return self._run(gen.exec_state, c, first=False)

    def _run(self, st, c: int, first: bool) -> float:
        lo, hi = st["cuts"][c], st["cuts"][c + 1]
        alpha = st["alpha"]
        # block table truncated to the tokens this chunk may attend: alpha + hi
        blocks, valid, need = [], [], alpha + hi
        for b, v in zip(st["blocks"], st["valid"]):
            if need <= 0:
                break
            blocks.append(b)
            valid.append(min(v, need))
            need -= v
        plan = kernels.AttnPlan([(hi - lo, alpha + lo, blocks, valid)],
                                block_tokens=self.pool.block_tokens,
                                n_q_heads=self.dims.shape.n_q_heads,
                                n_kv_heads=self.dims.shape.n_kv_heads, device=self.device)
        last = torch.tensor([hi - lo - 1], device=self.device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        fence = None
        if not first or self.swap_in == "modeled":
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
        self.last_logits = self.model.prefill(st["tok"][lo:hi], st["pos"][lo:hi],
                                              st["slots"][lo:hi], plan, last, layer_fence=fence)
        e1.record(self.stream)
        self.pool.wait_for(self.stream)  # later swap-outs read the finished pages
        e1.synchronize()
        self.chunks_run += 1
        return e0.elapsed_time(e1)


class ProfileExecutor:
    """Returns the engine profile's own interpolation: TimedEngine then reproduces
    ragsim.run exactly (the interception check)."""

    def __init__(self) -> None:
        from ragsim.cost_model import interpolate

        self.interpolate = interpolate
        self.last_ms = 0.0

    def on_admit(self, engine, gen, blocks, valid) -> None:
        self.last_ms = self.interpolate(engine.profile, gen.alpha, gen.beta)
