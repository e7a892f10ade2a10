"""The GPU hot path behind the reference's seams, as one batched server step.

A step serves a batch of requests the way a batching prefill server would:

  retrieval   staged exact top-k for the batch's query embeddings
              (tcgen05 scan, rcb_retrieval_topk) -> StagedRetrieval per request
  admission   for each request, the reference's tree decisions exactly as
              SimulationEngine._admit makes them (simulator.py:481-514):
              lookup -> pin -> evict_gpu -> load_to_gpu -> reserve_gpu; the
              TieredKnowledgeTree hooks turn every transition into a pool event
              (swap-out D2H / swap-in H2D on the copy stream, suffix blocks)
  prefill     per layer: RoPE + paged KV write of the suffix tokens, then
              prefix-aware attention over each request's block table
              (cached node pages + suffix pages)
  commit      SimulationEngine._commit's sequence (simulator.py:516-534):
              release_gpu -> insert_path (nodes adopt their suffix pages) ->
              update_node (PGDSF stats) -> unpin

Decisions only depend on the tree, so a step can be PLANNED on a shadow
(accounting-only) pool and REPLAYED later on the device pool: the allocator is
deterministic, so the planned block tables are the device pool's tables.  The
bench times replayed steps (device work only) and, separately, live steps
through the public API (host decisions + H2D/D2H included).
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels
from ._lib import RCB_SWAP_STAGED
from .cache import GenContext, TieredKnowledgeTree, _pool_call
from .pool import BlockPool, accounting_pool
from .workloads import ModelShape

from ragsim.policies import make_policy  # noqa: E402  (imported via .cache)
from ragsim.speculation import StagedRetrieval  # noqa: E402
from ragsim.tree import InsufficientEvictableCapacity, Tier  # noqa: E402


class EventLog:
    """Pool proxy that records events (planning on the shadow pool)."""

    EVENTS = ("node_alloc_gpu", "node_free_gpu", "node_free_host", "node_swap_out",
              "node_swap_in", "gen_reserve", "gen_free_segment", "node_adopt", "gen_release")

    def __init__(self, inner) -> None:
        self.inner = inner
        self.events: list[tuple] = []

    def __getattr__(self, name):
        target = getattr(self.inner, name)
        if name in self.EVENTS:
            def call(*args):
                self.events.append((name,) + tuple(list(a) if isinstance(a, (list, tuple)) else a
                                                   for a in args))
                return target(*args)
            return call
        return target

    def take(self) -> list[tuple]:
        ev, self.events = self.events, []
        return ev


def apply_events(pool: BlockPool, events) -> None:
    for ev in events:
        getattr(pool, ev[0])(*ev[1:])


@dataclass
class Admission:
    req_id: int
    docs: tuple
    prompt: int
    ctx: GenContext
    matched: list
    alpha: int
    beta: int
    swapped_in_tokens: int
    blocks: list = field(default_factory=list)
    valid: list = field(default_factory=list)


@dataclass
class StepPlan:
    admissions: list
    events: list  # pool events of the admission phase (replayable)
    commit_events: list
    # device buffers (filled by HotPath.prepare_device)
    dev: dict = field(default_factory=dict)

    @property
    def total_q(self) -> int:
        return sum(a.beta for a in self.admissions)


class HotPath:
    """Per-GPU replica: knowledge tree (reference decisions) + block pool + kernels."""

    def __init__(self, shape: ModelShape, *, gpu_capacity_tokens: int, host_capacity_tokens: int,
                 block_tokens: int, num_gpu_blocks: int, num_host_blocks: int, sizes,
                 profile, policy: str = "pgdsf", pool=None, device_pool: bool = True,
                 swap_mode: int = RCB_SWAP_STAGED, copy_stream=None,
                 indexed_leaves: bool = True) -> None:
        self.shape = shape
        self.sizes = sizes
        self.profile = profile
        self.block_tokens = block_tokens
        self.num_gpu_blocks = num_gpu_blocks
        if pool is None:
            if device_pool:
                pool = BlockPool(num_gpu_blocks, num_host_blocks, block_tokens=block_tokens,
                                 n_layers=shape.n_layers, n_kv_heads=shape.n_kv_heads,
                                 head_dim=shape.head_dim, swap_mode=swap_mode,
                                 copy_stream=copy_stream)
            else:
                pool = accounting_pool(num_gpu_blocks, num_host_blocks, block_tokens)
        self.pool = pool
        # indexed_leaves=False keeps the reference's linear victim scan (the CPU arm)
        self.tree = TieredKnowledgeTree(gpu_capacity_tokens, host_capacity_tokens,
                                        policy=make_policy(policy), pool=pool,
                                        indexed_leaves=indexed_leaves)
        self._keys = itertools.count()
        self._rope = None  # cos/sin table for RoPE fused into the attention kernel

    def rope_table(self, max_pos: int = 1 << 15) -> torch.Tensor:
        if self._rope is None or self._rope.shape[0] < max_pos:
            self._rope = kernels.rope_table(max_pos, self.shape.head_dim, self.shape.rope_theta)
        return self._rope

    # ------------------------------------------------------------------ decisions
    def admit(self, req_id: int, docs, prompt: int) -> Admission:
        """SimulationEngine._admit's sequence (simulator.py:481-514) for one request."""
        tree = self.tree
        match = tree.lookup(docs)
        miss = sum(self.sizes[d] for d in match.miss_docs)
        host_nodes = [n for n in match.matched_nodes if n.tier is Tier.HOST]
        promote = sum(n.size for n in host_nodes)
        need = promote + miss + prompt
        tree.pin(match.matched_nodes)
        try:
            if tree.gpu_free < need:
                tree.evict_gpu(need - tree.gpu_free)
        except InsufficientEvictableCapacity:
            tree.unpin(match.matched_nodes)
            raise
        ctx = GenContext(key=next(self._keys), seg_docs=list(match.miss_docs) + [None],
                         seg_tokens=[self.sizes[d] for d in match.miss_docs] + [prompt])
        tree.gen_ctx = ctx
        try:
            tree.load_to_gpu(host_nodes)
            tree.reserve_gpu(miss + prompt)
        finally:
            tree.gen_ctx = None
        adm = Admission(req_id, tuple(docs), prompt, ctx, list(match.matched_nodes),
                        match.hit_tokens, miss + prompt, promote)
        adm.blocks, adm.valid = self.pool.block_table([n.serial for n in adm.matched], ctx.key)
        return adm

    def commit(self, adm: Admission) -> None:
        """SimulationEngine._commit's sequence (simulator.py:516-534)."""
        tree = self.tree
        adm.ctx.phase = "commit"
        tree.gen_ctx = adm.ctx
        try:
            tree.release_gpu(adm.beta)
            path = tree.insert_path(adm.docs, [self.sizes[d] for d in adm.docs])
            cached = len(adm.matched)
            for i, node in enumerate(path):
                tree.update_node(node, i < cached, adm.alpha, adm.beta, self.profile)
            tree.unpin(adm.matched)
        finally:
            tree.gen_ctx = None
        _pool_call(self.pool.gen_release, adm.ctx.key)

    def admit_batch(self, batch) -> list[Admission]:
        """batch: [(req_id, docs, prompt)].  Stops early (returns a prefix) if the
        pinned batch exhausts evictable capacity; the caller defers the rest."""
        out = []
        for req_id, docs, prompt in batch:
            try:
                out.append(self.admit(req_id, docs, prompt))
            except InsufficientEvictableCapacity:
                break
        return out

    # ------------------------------------------------------------------ device plan
    def prepare_device(self, plan: StepPlan, device="cuda") -> None:
        """Upload the step's block tables, work list and suffix slot maps."""
        bt = self.block_tokens
        s = self.shape
        reqs = [(a.beta, a.alpha, a.blocks, a.valid) for a in plan.admissions]
        attn = kernels.AttnPlan(reqs, block_tokens=bt, n_q_heads=s.n_q_heads,
                                n_kv_heads=s.n_kv_heads, device=device)
        pos, slots, last = [], [], []
        q0 = 0
        for a in plan.admissions:
            nb_prefix = sum(-(-n.size // bt) for n in a.matched)
            seg_blocks = np.asarray(a.blocks[nb_prefix:], dtype=np.int64)
            seg_valid = np.asarray(a.valid[nb_prefix:], dtype=np.int64)
            if int(seg_valid.sum()) != a.beta:
                raise AssertionError("suffix segments do not cover beta tokens")
            # token t of the suffix -> pool slot block*bt + offset within its block
            starts = np.cumsum(seg_valid) - seg_valid
            off = np.arange(a.beta) - np.repeat(starts, seg_valid)
            slots.append(np.repeat(seg_blocks * bt, seg_valid) + off)
            pos.append(a.alpha + np.arange(a.beta))
            q0 += a.beta
            last.append(q0 - 1)
        pos = np.concatenate(pos) if pos else np.zeros(0, np.int64)
        slots = np.concatenate(slots) if slots else np.zeros(0, np.int64)
        arr = kernels._upload(np.concatenate([pos, slots, np.asarray(last, np.int64)])
                              .astype(np.int32), device)
        n = len(pos)
        plan.dev = {"attn": attn, "pos": arr[:n], "slots": arr[n:2 * n],
                    "last": arr[2 * n:].long(), "flops": attention_flops(self.shape, reqs)}

    def prefill(self, plan: StepPlan, qkv: torch.Tensor, q_rot, out: torch.Tensor,
                events=None, stream=None, layer_fence=None) -> None:
        """Launch KV-write + attention for every layer of the step (async).

        ``q_rot`` is unused (kept for callers of the pre-rotated path): Q's RoPE is
        applied inside the attention kernel from the hot path's cos/sin table.
        ``layer_fence(layer)`` (optional) runs before a layer's K/V write: with the step's
        swaps issued per layer group (BlockPool.flush_layered) the layer then waits only
        for its own group, i.e. for the swap-outs that read its slices of blocks the suffix
        now reuses and the swap-ins its attention reads."""
        s = self.shape
        d = plan.dev
        T = plan.total_q
        if T == 0:
            return
        if T > qkv.shape[0] or T > out.shape[0]:
            raise ValueError(f"step has {T} suffix tokens; activation buffers hold {qkv.shape[0]}")
        x = qkv[:T]
        q = x[:, : s.n_q_heads * s.head_dim]
        k = x[:, s.n_q_heads * s.head_dim:(s.n_q_heads + s.n_kv_heads) * s.head_dim]
        v = x[:, (s.n_q_heads + s.n_kv_heads) * s.head_dim:]
        o = out[:T]
        base = self.pool.gpu_base
        rope = self.rope_table(max(1 << 15, d["attn"].max_pos))
        for layer in range(s.n_layers):
            if layer_fence is not None:
                layer_fence(layer)
            # K/V: RoPE + paged write; Q's RoPE is fused into the attention kernel, which
            # reads the raw query columns of the QKV rows (no rotated-Q round trip)
            kernels.kv_write_rope(None, k, v, None, d["pos"], d["slots"], base,
                                  block_tokens=self.block_tokens, n_layers=s.n_layers,
                                  n_kv_heads=s.n_kv_heads, head_dim=s.head_dim, layer=layer,
                                  rope_theta=s.rope_theta, n_q_heads=s.n_q_heads, rope=rope,
                                  max_pos=d["attn"].max_pos, stream=stream)
            if events is not None:
                events[layer][0].record()
            kernels.prefix_prefill(q, o, d["attn"], base, self.num_gpu_blocks,
                                   block_tokens=self.block_tokens, n_layers=s.n_layers,
                                   n_kv_heads=s.n_kv_heads, head_dim=s.head_dim, layer=layer,
                                   rope=rope, n_q_heads=s.n_q_heads, stream=stream)
            if events is not None:
                events[layer][1].record()


def has_swaps(events) -> bool:
    """The step's pool events move bytes (a swap-out or a swap-in)."""
    return any(ev[0] in ("node_swap_out", "node_swap_in") for ev in events)


def attention_flops(shape: ModelShape, reqs) -> float:
    """Algorithmic FLOPs of one prefix-prefill launch (one layer): for each request
    4 * H_q * d_h * (alpha*beta + beta(beta+1)/2)."""
    tot = 0.0
    for beta, alpha, _, _ in reqs:
        tot += 4.0 * shape.n_q_heads * shape.head_dim * (alpha * beta + beta * (beta + 1) / 2.0)
    return tot


def staged_from_ids(ids_row: np.ndarray, interval_ms: float) -> StagedRetrieval:
    """One request's [S, k] staged ids -> the reference's StagedRetrieval (speculation.py:33-59)."""
    return StagedRetrieval(tuple(tuple(int(x) for x in st) for st in ids_row), interval_ms)
