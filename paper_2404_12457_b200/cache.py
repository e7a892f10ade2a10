"""Knowledge-tree tier transitions -> paged KV block pool.

The decision logic is the reference's, unchanged: ``TieredKnowledgeTree``
subclasses ragsim's ``KnowledgeTree`` (tree.py:131-571) and only OBSERVES
each transition after ``super()`` performs it, turning it into a block-pool
event.  ``TieredEngine`` subclasses ragsim's
``SimulationEngine`` (simulator.py:275-600), installs the tree where the
reference builds its own (simulator.py:291-296), and gives the tree the
generation context of admit / commit / abort (simulator.py:481-559) so
suffix blocks can be reserved, adopted by the nodes insert_path creates, and
released.  The pool may be the native ``BlockPool`` (product) or the Python
``BlockOracle`` (tests): both expose the same event methods.

Transition map:
  _demote_from_gpu (tree.py:450-473): first eviction -> node_swap_out;
      repeat eviction (host copy kept) -> node_free_gpu; host full -> drop:
      node_free_gpu + node_free_host of the host descendants (_drop_subtree :482-502)
  _free_from_host (tree.py:475-480)  -> node_free_host
  load_to_gpu (tree.py:296-318)      -> node_swap_in (host copy retained)
  reserve_gpu in _admit (:320-327)   -> gen_reserve(one segment per miss doc + prompt)
  release_gpu in _commit (:329-333)  -> gen_free_segment(prompt)
  insert_path node creation (:252-294) -> node_adopt(segment of that doc), or
      node_alloc_gpu when no generation supplies the KV; an existing node makes
      the generation's segment a duplicate -> gen_free_segment
  release_gpu in _abort (simulator.py:549-559) -> gen_release
"""

from __future__ import annotations

import heapq
import itertools
from dataclasses import dataclass, field

from ._ragsim import import_ragsim
from .pool import PoolCapacityError

_ragsim = import_ragsim()
from ragsim.policies import make_policy  # noqa: E402
from ragsim.simulator import SimulationEngine  # noqa: E402
from ragsim.tree import CacheError, KnowledgeTree, Tier  # noqa: E402


class BlockPoolExhausted(CacheError):
    """The pool ran out of blocks although the tree's token accounting fit:
    a pool-sizing bug, never a normal admission stall."""


@dataclass
class GenContext:
    key: int
    seg_docs: list  # doc id per segment; None for the prompt segment
    seg_tokens: list
    phase: str = "admit"
    seg_of_doc: dict = field(default_factory=dict)

    def __post_init__(self) -> None:
        self.seg_of_doc = {d: i for i, d in enumerate(self.seg_docs) if d is not None}

    @property
    def prompt_seg(self) -> int:
        return len(self.seg_docs) - 1


def _pool_call(fn, *args):
    try:
        return fn(*args)
    except CacheError:
        raise
    except Exception as exc:  # PoolCapacityError / the oracle's capacity error / PoolError
        if isinstance(exc, PoolCapacityError) or type(exc).__name__ == "OracleCapacityError":
            raise BlockPoolExhausted(str(exc)) from exc
        raise CacheError(str(exc)) from exc


class _IndexedLeaves(set):
    """The reference's tier-leaf set plus a lazy min-heap on the policy's eviction key.

    ``KnowledgeTree._min_leaf`` (tree.py:407-411) scans every leaf per victim: with a
    1.1M-token GPU tier that scan is ~85% of the host time of a step.  The eviction key
    (priority, -size, doc, serial) (policies.py:46-50) ends in the node's unique serial, so
    it is a total order and the heap minimum is exactly the victim ``min()`` picks.  The
    reference mutates the set with add/discard only; keys change only in update_node
    (tree.py:233-246), which re-pushes the node.  Stale entries (left the set, or an old
    key) are dropped when they surface."""

    def __init__(self, items, key) -> None:
        super().__init__(items)
        self.key = key
        self.heap: list = []
        self._seq = itertools.count()
        for node in items:
            self.push(node)

    def push(self, node) -> None:
        heapq.heappush(self.heap, (self.key(node), next(self._seq), node))

    def add(self, node) -> None:
        if node not in self:
            super().add(node)
            self.push(node)

    def min_unpinned(self):
        heap, aside, found = self.heap, [], None
        while heap:
            k, _, node = heap[0]
            if node not in self or k != self.key(node):
                heapq.heappop(heap)
            elif node.pinned:
                aside.append(heapq.heappop(heap))
            else:
                found = node
                break
        for entry in aside:
            heapq.heappush(heap, entry)
        if len(heap) > 64 and len(heap) > 4 * len(self):
            self.heap = [(self.key(n), next(self._seq), n) for n in self]
            heapq.heapify(self.heap)
        return found


class TieredKnowledgeTree(KnowledgeTree):
    """ragsim KnowledgeTree whose tier transitions drive a block pool."""

    def __init__(self, gpu_capacity: int, host_capacity: int, policy=None,
                 frequency_decay: float = 1.0, *, pool, indexed_leaves: bool = True) -> None:
        super().__init__(gpu_capacity, host_capacity, policy=policy,
                         frequency_decay=frequency_decay)
        self.pool = pool
        self.gen_ctx: GenContext | None = None
        if indexed_leaves:
            self._gpu_leaves = _IndexedLeaves(self._gpu_leaves, self.policy.eviction_key)
            self._host_leaves = _IndexedLeaves(self._host_leaves, self.policy.eviction_key)

    # -- victim selection (same victims as tree.py:407-411, without the scan) -------
    def _min_leaf(self, leaves):
        if isinstance(leaves, _IndexedLeaves):
            return leaves.min_unpinned()
        return super()._min_leaf(leaves)

    def update_node(self, node, *args, **kwargs) -> None:
        super().update_node(node, *args, **kwargs)
        for leaves in (self._gpu_leaves, self._host_leaves):
            if isinstance(leaves, _IndexedLeaves) and node in leaves:
                leaves.push(node)

    # -- eviction side ------------------------------------------------------
    def _demote_from_gpu(self, node) -> None:
        had_copy = node.has_host_copy
        super()._demote_from_gpu(node)
        if had_copy:
            _pool_call(self.pool.node_free_gpu, node.serial)  # swap-out-only-once: no copy
        elif node.tier is Tier.HOST:
            _pool_call(self.pool.node_swap_out, [node.serial])
        else:  # dropped outright (host could not absorb it)
            _pool_call(self.pool.node_free_gpu, node.serial)

    def _drop_subtree(self, node) -> None:
        doomed = []
        stack = list(node.children.values())
        while stack:
            child = stack.pop()
            stack.extend(child.children.values())
            if child.tier is Tier.HOST:
                doomed.append(child.serial)
        super()._drop_subtree(node)
        for serial in doomed:
            _pool_call(self.pool.node_free_host, serial)

    def _free_from_host(self, node) -> None:
        super()._free_from_host(node)
        _pool_call(self.pool.node_free_host, node.serial)

    # -- promotion / reservation side -------------------------------------
    def load_to_gpu(self, nodes) -> int:
        promoted = [n for n in nodes if n.tier is Tier.HOST]
        try:
            return super().load_to_gpu(nodes)
        finally:
            moved = [n.serial for n in promoted if n.tier is Tier.GPU]
            if moved:
                _pool_call(self.pool.node_swap_in, moved)

    def reserve_gpu(self, tokens: int) -> None:
        super().reserve_gpu(tokens)
        ctx = self.gen_ctx
        if ctx is not None and ctx.phase == "admit":
            _pool_call(self.pool.gen_reserve, ctx.key, ctx.seg_tokens)

    def release_gpu(self, tokens: int) -> None:
        super().release_gpu(tokens)
        ctx = self.gen_ctx
        if ctx is None:
            return
        if ctx.phase == "commit":
            _pool_call(self.pool.gen_free_segment, ctx.key, ctx.prompt_seg)
        elif ctx.phase == "abort":
            _pool_call(self.pool.gen_release, ctx.key)

    def insert_path(self, doc_sequence, sizes):
        if len(doc_sequence) != len(sizes):
            return super().insert_path(doc_sequence, sizes)  # raises like the reference
        # Extend one document at a time: each call re-walks (and re-pins) the
        # existing prefix exactly as a single call would, so decisions are
        # identical, and the creation of node i can be observed in order.
        ctx = self.gen_ctx if (self.gen_ctx is not None and self.gen_ctx.phase == "commit") else None
        path = []
        for i in range(len(doc_sequence)):
            before = self._node_serial
            path = super().insert_path(doc_sequence[: i + 1], sizes[: i + 1])
            node = path[-1]
            seg = ctx.seg_of_doc.get(doc_sequence[i]) if ctx is not None else None
            if self._node_serial != before:
                if seg is not None:
                    _pool_call(self.pool.node_adopt, node.serial, ctx.key, seg)
                else:
                    _pool_call(self.pool.node_alloc_gpu, node.serial, node.size)
            elif seg is not None:
                _pool_call(self.pool.gen_free_segment, ctx.key, seg)
        return path


class TieredEngine(SimulationEngine):
    """ragsim SimulationEngine with a TieredKnowledgeTree and an optional GPU
    executor that runs each admitted generation's prefill on the block table.

    Decisions, timing and the report are the reference's (virtual clock driven
    by the cost profile — the "parity mode" of SURVEY H1)."""

    def __init__(self, config, trace, sizes, stage_provider=None, *, pool, executor=None,
                 record_tables: bool = False) -> None:
        super().__init__(config, trace, sizes, stage_provider=stage_provider)
        self.tree = TieredKnowledgeTree(
            config.gpu_capacity_tokens,
            config.host_capacity_tokens,
            policy=make_policy(config.policy),
            frequency_decay=config.frequency_decay,
            pool=pool,
        )
        self.pool = pool
        self.executor = executor
        self._gen_keys = itertools.count()
        self.record_tables = record_tables
        self.tables: list[tuple] = []  # (gen key, request id, node serials, blocks, valid)

    def _admit(self, gen) -> None:
        match = self.tree.lookup(gen.docs)
        seg_docs = list(match.miss_docs) + [None]
        seg_tokens = [self.sizes[d] for d in match.miss_docs] + [gen.request.prompt_tokens]
        ctx = GenContext(key=next(self._gen_keys), seg_docs=seg_docs, seg_tokens=seg_tokens)
        self.tree.gen_ctx = ctx
        try:
            super()._admit(gen)
        finally:
            self.tree.gen_ctx = None
        gen.pool_ctx = ctx
        if self.record_tables or self.executor is not None:
            serials = [n.serial for n in gen.matched_nodes]
            blocks, valid = self.pool.block_table(serials, ctx.key)
            if self.record_tables:
                self.tables.append((ctx.key, gen.request.id, serials, blocks, valid))
            if self.executor is not None:
                self.executor.on_admit(self, gen, blocks, valid)

    def _commit(self, gen) -> None:
        ctx = gen.pool_ctx
        ctx.phase = "commit"
        self.tree.gen_ctx = ctx
        try:
            super()._commit(gen)
        finally:
            self.tree.gen_ctx = None
        _pool_call(self.pool.gen_release, ctx.key)

    def _abort(self, gen) -> None:
        ctx = getattr(gen, "pool_ctx", None)
        if ctx is not None and gen.reserved:
            ctx.phase = "abort"
            self.tree.gen_ctx = ctx
        try:
            super()._abort(gen)
        finally:
            self.tree.gen_ctx = None


def run_tiered(config, trace, sizes, *, pool, stage_provider=None, executor=None,
               record_tables: bool = False):
    """ragsim.run with the block pool attached; returns (SimReport, engine)."""
    engine = TieredEngine(config, trace, sizes, stage_provider=stage_provider, pool=pool,
                          executor=executor, record_tables=record_tables)
    return engine.run(), engine
