"""GPU block pool under the reference engine: bytes survive every tier transition.

The unmodified ragsim engine (desk recipes of tests/golden) drives the native
pool with real HBM + pinned host memory.  Each admitted generation's suffix
segments are filled (on the compute stream, fenced against the copy stream,
SURVEY H3) with a pattern keyed by the node's document PATH (a node's KV
depends on its prefix).  After the run every node's GPU
blocks and host copy must hold exactly its pattern — bit-exact through
swap-out (D2H), swap-in (H2D), zero-copy drops and block reuse — and the
block tables must equal the golden ones.
"""

import gzip
import json
import os
import zlib

import numpy as np
import pytest
import torch

from oracle.block_oracle import EventRecorder, replay
from paper_2404_12457_b200 import _lib
from paper_2404_12457_b200._ragsim import ragsim_available
from paper_2404_12457_b200.pool import BlockPool

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GEOM = dict(block_tokens=16, n_layers=2, n_kv_heads=4, head_dim=64)  # tiny model: 32 KB blocks
MODES = [_lib.RCB_SWAP_STAGED, _lib.RCB_SWAP_ZEROCOPY, _lib.RCB_SWAP_DMA]


def load(name):
    with gzip.open(os.path.join(HERE, "golden", name), "rt") as fp:
        return json.load(fp)


def pattern(path, j, nbytes):
    h = zlib.crc32(repr(tuple(path)).encode())
    mult = (h % 127) * 2 + 1
    add = ((h >> 8) + 31 * j) % 256
    return ((np.arange(nbytes, dtype=np.int64) * mult + add) % 256).astype(np.uint8)


class FillExecutor:
    """Writes each new segment's 'KV' on the compute stream."""

    def __init__(self, pool, pool_u8):
        self.pool = pool
        self.u8 = pool_u8
        self.stream = torch.cuda.current_stream()

    def on_admit(self, engine, gen, blocks, valid):
        ctx = gen.pool_ctx
        self.pool.fence_into(self.stream)  # swap copies done before blocks are rewritten
        n_hit = len(gen.matched_nodes)
        for seg, doc in enumerate(ctx.seg_docs):
            if doc is None:
                continue  # prompt segment is never cached
            path = list(gen.docs[: n_hit + seg + 1])
            assert path[-1] == doc
            for j, b in enumerate(self.pool.gen_blocks(ctx.key, seg)):
                self.u8[b].copy_(torch.from_numpy(pattern(path, j, self.u8.shape[1])),
                                 non_blocking=False)
        self.pool.wait_for(self.stream)  # later swap-outs read the finished writes


def _node_path(node):
    path = []
    while node is not None and node.parent is not None:
        path.append(node.doc)
        node = node.parent
    return path[::-1]


@pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("golden", ["desk_c8.json.gz", "desk_drop_lru.json.gz"])
def test_engine_bytes_roundtrip(golden, mode):
    import dataclasses

    from ragsim.config import RunConfig

    from paper_2404_12457_b200 import cache
    from tests.golden.make_golden import desk_trace

    g = load(golden)
    r = g["recipe"]
    trace, sizes = desk_trace(r["seed"], r["duration_s"], r["rate"], r["pool"])
    fields = {f.name for f in dataclasses.fields(RunConfig)}
    cfg = RunConfig(**{k: (tuple(v) if isinstance(v, list) else v)
                       for k, v in g["config"].items() if k in fields})
    ng, nh = g["num_gpu_blocks"], g["num_host_blocks"]
    bb = 2 * GEOM["n_layers"] * GEOM["n_kv_heads"] * GEOM["block_tokens"] * GEOM["head_dim"] * 2
    pool_u8 = torch.zeros((ng, bb), dtype=torch.uint8, device="cuda")
    pool = BlockPool(ng, nh, swap_mode=mode, gpu_base=pool_u8.data_ptr(), **GEOM)
    rec = EventRecorder(pool)
    report, engine = cache.run_tiered(cfg, trace, sizes, pool=rec, record_tables=True,
                                      executor=FillExecutor(pool, pool_u8))
    pool.sync()
    torch.cuda.synchronize()
    assert json.loads(json.dumps(rec.events)) == g["events"]
    host = pool.host_view()
    gpu = pool_u8.cpu().numpy()
    checked = 0
    for node in engine.tree.nodes():
        path = _node_path(node)
        if node.tier.value == "gpu":
            for j, b in enumerate(pool.node_blocks(node.serial, 0)):
                assert np.array_equal(gpu[b], pattern(path, j, bb)), f"GPU bytes of {path}"
                checked += 1
        if node.has_host_copy:
            for j, b in enumerate(pool.node_blocks(node.serial, 1)):
                assert np.array_equal(host[b], pattern(path, j, bb)), f"host bytes of {path}"
                checked += 1
    assert checked > 100
    st = pool.stats()
    assert st["swap_out_blocks"] > 0 and st["swap_in_blocks"] > 0
    pool.close()


@pytest.mark.parametrize("mode", MODES)
def test_replay_golden_on_device_pool(mode):
    g = load("desk_c8.json.gz")
    pool = BlockPool(g["num_gpu_blocks"], g["num_host_blocks"], swap_mode=mode, **GEOM)
    assert replay(g["events"], pool) == 380
    pool.sync()
    st = pool.stats()
    assert st["d2h_bytes"] == st["swap_out_blocks"] * pool.block_bytes
    pool.close()
