"""The indexed leaf heap picks exactly the reference's victims.

``TieredKnowledgeTree`` replaces the linear ``_min_leaf`` scan (ragsim
tree.py:407-411) with a lazy heap on the policy's eviction key.  Here the
unmodified reference ``KnowledgeTree`` and the indexed subclass are driven by
the same random operation stream (inserts, accesses, pins, GPU/host
evictions, swap-ins) for every policy; victims, exceptions and the full tree
snapshot must agree after every operation.
"""

import numpy as np
import pytest

from paper_2404_12457_b200._ragsim import ragsim_available

pytestmark = pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")


class _NullPool:
    def __getattr__(self, name):
        return lambda *a, **k: None


def _drive(tree, rng_seed, n_ops, docs, sizes):
    from ragsim.cost_model import synthetic_profile
    from ragsim.tree import CacheError

    rng = np.random.default_rng(rng_seed)
    profile = synthetic_profile()
    log = []
    pinned = []
    for _ in range(n_ops):
        op = rng.integers(0, 6)
        seq = [int(d) for d in rng.choice(docs, size=int(rng.integers(1, 4)), replace=False)]
        try:
            if op == 0:
                path = tree.insert_path(seq, [sizes[d] for d in seq])
                log.append(("ins", [n.serial for n in path]))
            elif op == 1:
                m = tree.lookup(seq)
                for n in m.matched_nodes:
                    tree.update_node(n, bool(rng.integers(0, 2)), int(rng.integers(0, 2048)),
                                     int(rng.integers(1, 2048)), profile)
                log.append(("upd", [n.serial for n in m.matched_nodes]))
            elif op == 2:
                m = tree.lookup(seq)
                if m.matched_nodes:
                    tree.pin(m.matched_nodes)
                    pinned.append(m.matched_nodes)
                if len(pinned) > 3 or (pinned and rng.integers(0, 2)):
                    tree.unpin(pinned.pop(0))
                log.append(("pin", len(pinned)))
            elif op == 3:
                v = tree.evict_gpu(int(rng.integers(1, 1500)))
                log.append(("evg", [n.serial for n in v]))
            elif op == 4:
                v = tree.evict_host(int(rng.integers(1, 1500)))
                log.append(("evh", [n.serial for n in v]))
            else:
                m = tree.lookup(seq)
                host = [n for n in m.matched_nodes if n.tier.name == "HOST"]
                need = sum(n.size for n in host)
                if host and tree.gpu.free < need:
                    tree.evict_gpu(need - tree.gpu.free)
                log.append(("load", tree.load_to_gpu(m.matched_nodes) if host else 0))
        except CacheError as exc:
            log.append(("err", type(exc).__name__))
        log.append(("snap", tree.snapshot()))
    return log


@pytest.mark.parametrize("policy", ["pgdsf", "gdsf", "lru", "lfu"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_indexed_victims_match_reference(policy, seed):
    from ragsim.policies import make_policy
    from ragsim.tree import KnowledgeTree

    from paper_2404_12457_b200.cache import TieredKnowledgeTree

    rng = np.random.default_rng(100 + seed)
    docs = np.arange(40)
    sizes = {int(d): int(rng.choice([64, 128, 200, 512])) for d in docs}
    # equal sizes and priorities are common: the key's serial must break the ties
    ref = KnowledgeTree(4096, 6000, policy=make_policy(policy))
    ours = TieredKnowledgeTree(4096, 6000, policy=make_policy(policy), pool=_NullPool())
    a = _drive(ref, seed, 600, docs, sizes)
    b = _drive(ours, seed, 600, docs, sizes)
    assert a == b
    assert sum(1 for e in a if e[0] in ("evg", "evh") and e[1]) > 20
    ours.check_invariants()
