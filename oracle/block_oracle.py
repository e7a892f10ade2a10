"""ORACLE (test infrastructure only — never imported by the product path).

Pure-Python restatement of the block allocator behind the knowledge tree's
tier transitions.  ragsim tracks tokens, not blocks, so block
tables are a NEW concept with no reference golden; this
oracle defines them from the reference's own event stream:

* every tier transition of ragsim's KnowledgeTree maps to one event
  (tree.py:296-318 load_to_gpu -> swap_in; :320-333 reserve/release ->
  gen_reserve / gen_free_segment / gen_release; :252-294 insert_path node
  creation -> node_adopt; :450-473 _demote_from_gpu -> swap_out or, with a
  host copy already present, free_gpu; :475-480 _free_from_host -> free_host;
  :482-502 _drop_subtree -> free_gpu + free_host of host descendants);
* nodes are block-aligned: ceil(tokens / block_tokens) blocks each;
* both tiers allocate lowest-free-block-first (a min-heap).

It is pinned by construction against ragsim: the event stream it consumes
is produced by the unmodified reference tree, and tests check that the
reference's own accounting (gpu.used / host.used, tree.py:57-67) is
reproduced token-for-token by the blocks it hands out.
"""

from __future__ import annotations

import heapq


class OracleCapacityError(RuntimeError):
    pass


class BlockOracle:
    def __init__(self, num_gpu_blocks: int, num_host_blocks: int, block_tokens: int) -> None:
        self.bt = block_tokens
        self.gpu_free = list(range(num_gpu_blocks))
        self.host_free = list(range(num_host_blocks))
        heapq.heapify(self.gpu_free)
        heapq.heapify(self.host_free)
        self.nodes: dict[int, dict] = {}  # key -> {"tokens", "gpu": [...], "host": [...]}
        self.gens: dict[int, list[dict]] = {}  # gen -> [{"tokens", "blocks", "done"}]
        self.log: list[tuple] = []

    def _nb(self, tokens: int) -> int:
        return -(-tokens // self.bt)

    @staticmethod
    def _take(heap: list[int], n: int) -> list[int]:
        if len(heap) < n:
            raise OracleCapacityError(f"need {n} blocks, {len(heap)} free")
        return [heapq.heappop(heap) for _ in range(n)]

    @staticmethod
    def _give(heap: list[int], blocks: list[int]) -> None:
        for b in blocks:
            heapq.heappush(heap, b)

    # ------------------------------------------------------------------ events
    def node_alloc_gpu(self, key: int, tokens: int) -> None:
        self.log.append(("alloc", key, tokens))
        node = self.nodes.setdefault(key, {"tokens": tokens, "gpu": [], "host": []})
        assert not node["gpu"]
        node["tokens"] = tokens
        node["gpu"] = self._take(self.gpu_free, self._nb(tokens))

    def node_free_gpu(self, key: int) -> None:
        self.log.append(("free_gpu", key))
        node = self.nodes[key]
        assert node["gpu"], "node not GPU-resident"
        self._give(self.gpu_free, node["gpu"])
        node["gpu"] = []
        if not node["host"]:
            del self.nodes[key]

    def node_free_host(self, key: int) -> None:
        self.log.append(("free_host", key))
        node = self.nodes[key]
        assert node["host"], "node has no host copy"
        self._give(self.host_free, node["host"])
        node["host"] = []
        if not node["gpu"]:
            del self.nodes[key]

    def node_swap_out(self, keys) -> None:
        self.log.append(("swap_out", tuple(keys)))
        need = sum(self._nb(self.nodes[k]["tokens"]) for k in keys)
        if len(self.host_free) < need:
            raise OracleCapacityError("out of host blocks")
        for k in keys:
            node = self.nodes[k]
            assert node["gpu"] and not node["host"]
            node["host"] = self._take(self.host_free, self._nb(node["tokens"]))
            self._give(self.gpu_free, node["gpu"])
            node["gpu"] = []

    def node_swap_in(self, keys) -> None:
        self.log.append(("swap_in", tuple(keys)))
        need = sum(self._nb(self.nodes[k]["tokens"]) for k in keys)
        if len(self.gpu_free) < need:
            raise OracleCapacityError("out of GPU blocks")
        for k in keys:
            node = self.nodes[k]
            assert node["host"] and not node["gpu"]
            node["gpu"] = self._take(self.gpu_free, self._nb(node["tokens"]))

    def gen_reserve(self, gen: int, seg_tokens) -> None:
        self.log.append(("reserve", gen, tuple(seg_tokens)))
        need = sum(self._nb(t) for t in seg_tokens)
        if len(self.gpu_free) < need:
            raise OracleCapacityError("out of GPU blocks")
        assert gen not in self.gens
        self.gens[gen] = [{"tokens": t, "blocks": self._take(self.gpu_free, self._nb(t)),
                           "done": False} for t in seg_tokens]

    def gen_free_segment(self, gen: int, seg: int) -> None:
        self.log.append(("free_seg", gen, seg))
        s = self.gens[gen][seg]
        assert not s["done"]
        self._give(self.gpu_free, s["blocks"])
        s["blocks"] = []
        s["done"] = True

    def node_adopt(self, key: int, gen: int, seg: int) -> None:
        self.log.append(("adopt", key, gen, seg))
        s = self.gens[gen][seg]
        assert not s["done"]
        node = self.nodes.setdefault(key, {"tokens": s["tokens"], "gpu": [], "host": []})
        assert not node["gpu"]
        node["tokens"] = s["tokens"]
        node["gpu"] = s["blocks"]
        s["blocks"] = []
        s["done"] = True

    def gen_release(self, gen: int) -> None:
        self.log.append(("release", gen))
        for s in self.gens.pop(gen):
            if not s["done"]:
                self._give(self.gpu_free, s["blocks"])

    # ------------------------------------------------------------------ queries
    def node_blocks(self, key: int, tier: int = 0) -> list[int]:
        node = self.nodes.get(key)
        if node is None:
            return []
        return list(node["gpu"] if tier == 0 else node["host"])

    def block_table(self, node_keys, gen: int = -1) -> tuple[list[int], list[int]]:
        blocks: list[int] = []
        valid: list[int] = []

        def push(bl, tokens):
            for i, b in enumerate(bl):
                blocks.append(b)
                valid.append(self.bt if i + 1 < len(bl) else tokens - i * self.bt)

        for k in node_keys:
            node = self.nodes[k]
            assert node["gpu"], "block table node not GPU-resident"
            push(node["gpu"], node["tokens"])
        if gen >= 0:
            for s in self.gens[gen]:
                assert not s["done"]
                push(s["blocks"], s["tokens"])
        return blocks, valid

    # no device work in the oracle
    def flush(self) -> None:
        pass


class EventRecorder:
    """Forwards pool events to ``inner`` and records them, plus every block
    table the engine reads, as a replayable list (golden fixtures)."""

    EVENTS = ("node_alloc_gpu", "node_free_gpu", "node_free_host", "node_swap_out",
              "node_swap_in", "gen_reserve", "gen_free_segment", "node_adopt", "gen_release")

    def __init__(self, inner) -> None:
        self.inner = inner
        self.events: list[list] = []

    def __getattr__(self, name):
        target = getattr(self.inner, name)
        if name in self.EVENTS:
            def call(*args):
                self.events.append([name] + [list(a) if isinstance(a, (list, tuple)) else a
                                             for a in args])
                return target(*args)
            return call
        return target

    def block_table(self, node_keys, gen: int = -1):
        blocks, valid = self.inner.block_table(node_keys, gen)
        self.events.append(["block_table", list(node_keys), gen, list(blocks), list(valid)])
        return blocks, valid


def replay(events, pool) -> int:
    """Drive ``pool`` with a recorded event list; assert every recorded block
    table is reproduced.  Returns the number of tables checked."""
    checked = 0
    for ev in events:
        name, args = ev[0], ev[1:]
        if name == "block_table":
            keys, gen, blocks, valid = args
            got = pool.block_table(keys, gen)
            assert list(got[0]) == blocks and list(got[1]) == valid, f"table mismatch at {ev}"
            checked += 1
        else:
            getattr(pool, name)(*args)
    return checked
