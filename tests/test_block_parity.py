"""Block tables and tier-transition sequences: bit-exact parity.

Golden fixtures (tests/golden/*.json.gz) were generated FROM THE REFERENCE by
tests/golden/make_golden.py: the unmodified ragsim engine drives the
transition hooks; the Python block oracle turns them into block tables.
Here the native pool (C++ allocator, accounting mode — no GPU needed)
replays the same event streams and must reproduce every table; with ragsim
importable, the live engine is re-run and must reproduce the reference's
report byte-for-byte and the golden event stream exactly.
"""

import dataclasses
import glob
import gzip
import json
import os

import pytest

from oracle.block_oracle import BlockOracle, EventRecorder, replay
from paper_2404_12457_b200 import pool as pool_mod
from paper_2404_12457_b200._ragsim import ragsim_available

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "desk_*.json.gz")))


def load(path):
    with gzip.open(path, "rt") as fp:
        return json.load(fp)


@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_oracle_replay_reproduces_golden(path):
    g = load(path)
    orc = BlockOracle(g["num_gpu_blocks"], g["num_host_blocks"], g["block_tokens"])
    n = replay(g["events"], orc)
    assert n == sum(1 for e in g["events"] if e[0] == "block_table") and n > 0
    for serial, node in g["nodes"].items():
        assert orc.node_blocks(int(serial), 0) == node["gpu"]
        assert orc.node_blocks(int(serial), 1) == node["host"]


@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_native_pool_replay_matches_golden(path):
    g = load(path)
    p = pool_mod.accounting_pool(g["num_gpu_blocks"], g["num_host_blocks"], g["block_tokens"])
    replay(g["events"], p)
    for serial, node in g["nodes"].items():
        assert p.node_blocks(int(serial), pool_mod.GPU) == node["gpu"]
        assert p.node_blocks(int(serial), pool_mod.HOST) == node["host"]
    st = p.stats()
    swapped = sum(len(e[1]) for e in g["events"] if e[0] == "node_swap_out")
    assert st["swap_out_calls"] == sum(1 for e in g["events"] if e[0] == "node_swap_out")
    assert swapped == g["aggregates"]["swap_outs"]


def test_golden_accounting_matches_reference_tokens():
    for path in GOLDEN:
        g = load(path)
        bt = g["block_tokens"]
        gpu_nodes = [n for n in g["nodes"].values() if n["tier"] == "gpu"]
        for n in g["nodes"].values():
            nb = -(-n["tokens"] // bt)
            assert len(n["gpu"]) in (0, nb) and len(n["host"]) in (0, nb)
            assert (len(n["gpu"]) > 0) == (n["tier"] == "gpu")
        # every GPU block is owned once
        owned = [b for n in gpu_nodes for b in n["gpu"]]
        assert len(owned) == len(set(owned))


def test_native_pool_errors_map_to_capacity():
    p = pool_mod.accounting_pool(4, 2, 16)
    p.node_alloc_gpu(1, 64)
    with pytest.raises(pool_mod.PoolCapacityError):
        p.node_alloc_gpu(2, 1)
    with pytest.raises(pool_mod.PoolCapacityError):
        p.node_swap_out([1])  # needs 4 host blocks, 2 exist
    with pytest.raises(pool_mod.PoolError):
        p.node_free_host(1)


def test_lowest_free_first_both_implementations():
    orc = BlockOracle(16, 8, 16)
    nat = pool_mod.accounting_pool(16, 8, 16)
    ops = [("node_alloc_gpu", 1, 40), ("node_alloc_gpu", 2, 16), ("node_free_gpu", 1),
           ("gen_reserve", 0, [20, 5]), ("node_swap_out", [2]), ("node_adopt", 3, 0, 0),
           ("gen_free_segment", 0, 1), ("gen_release", 0), ("node_swap_in", [2])]
    for op in ops:
        getattr(orc, op[0])(*op[1:])
        getattr(nat, op[0])(*op[1:])
    for key in (2, 3):
        for tier in (0, 1):
            assert orc.node_blocks(key, tier) == nat.node_blocks(key, tier)
    assert orc.node_blocks(3, 0) == [0, 1]  # seg 0 (20 tokens) took the two lowest
    assert orc.node_blocks(2, 1) == [0]


needs_ragsim = pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")


@needs_ragsim
@pytest.mark.parametrize("path", GOLDEN, ids=os.path.basename)
def test_live_engine_reproduces_reference_and_golden(path):
    from ragsim.config import RunConfig
    from ragsim.simulator import run

    from paper_2404_12457_b200 import cache
    from tests.golden.make_golden import desk_trace

    g = load(path)
    r = g["recipe"]
    trace, sizes = desk_trace(r["seed"], r["duration_s"], r["rate"], r["pool"])
    fields = {f.name for f in dataclasses.fields(RunConfig)}
    cfgd = {k: (tuple(v) if isinstance(v, list) else v) for k, v in g["config"].items()
            if k in fields}
    cfg = RunConfig(**cfgd)
    plain = run(cfg, trace, sizes)
    nat = pool_mod.accounting_pool(g["num_gpu_blocks"], g["num_host_blocks"], g["block_tokens"])
    rec = EventRecorder(nat)
    report, _ = cache.run_tiered(cfg, trace, sizes, pool=rec, record_tables=True)
    assert report.to_json(cfg) == plain.to_json(cfg)
    assert report.per_request_csv() == plain.per_request_csv()
    assert json.loads(json.dumps(rec.events)) == g["events"]
    assert report.aggregates()["swap_outs"] == g["aggregates"]["swap_outs"]


def test_native_pool_rejects_duplicate_keys_without_mutation():
    # a key repeated in one swap call would leak blocks and alias a host copy: the C-ABI
    # rejects the call before touching any state (block_pool.cpp has_duplicate)
    p = pool_mod.accounting_pool(8, 8, 16)
    p.node_alloc_gpu(1, 32)
    gpu_before = p.node_blocks(1, pool_mod.GPU)
    with pytest.raises(pool_mod.PoolError):
        p.node_swap_out([1, 1])
    assert p.node_blocks(1, pool_mod.GPU) == gpu_before
    p.node_swap_out([1])  # demotes: host copy made, GPU blocks freed
    host = p.node_blocks(1, pool_mod.HOST)
    assert len(host) == 2 and p.node_blocks(1, pool_mod.GPU) == []
    with pytest.raises(pool_mod.PoolError):
        p.node_swap_in([1, 1])
    assert p.node_blocks(1, pool_mod.HOST) == host
    p.node_swap_in([1])
    assert len(p.node_blocks(1, pool_mod.GPU)) == 2


def test_pool_blocks_counts_node_tails_when_any_doc_is_ragged():
    from paper_2404_12457_b200.workloads import pool_blocks
    # every doc a multiple of the block: no tail blocks, just ceil(cap/B) + segments + slack
    assert pool_blocks(10240, 16, [16, 32, 64], 4) == 640 + 4 + 8
    # one ragged doc (17 tokens): up to cap // min_doc resident nodes may each own a tail block
    assert pool_blocks(10240, 16, [16, 17, 64], 4) == 640 + 10240 // 16 + 4 + 8
    assert pool_blocks(0, 16, [17], 4) == 0
