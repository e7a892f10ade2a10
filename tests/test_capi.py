"""The C-ABI library loads and exports every symbol include/ragcache_b200.h declares."""

import os
import re

from paper_2404_12457_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ragcache_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rcb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"


def test_bindings_cover_header_exactly():
    bound = sorted(n for n, _, _ in _lib.SIGNATURES)
    assert bound == header_functions()


def test_version_and_error_plumbing():
    lib = _lib.load()
    assert lib.rcb_version() >= 1
    # argument errors surface through rcb_last_error without touching a GPU
    code = lib.rcb_kv_block_copy(None, None, 7, None, 1, None)
    assert code == _lib.RCB_ERR_ARG
    assert b"multiple of 16" in lib.rcb_last_error()


def test_attn_plan_host_logic():
    import numpy as np

    from paper_2404_12457_b200 import kernels

    # two requests: a cached 1024-token prefix + 32 prompt tokens, and a full miss
    reqs = [(32, 1024, list(range(66)), [16] * 66), (544, 0, list(range(34)), [16] * 34)]
    plan = kernels.AttnPlan(reqs, block_tokens=16, n_q_heads=32, n_kv_heads=8, device="cpu")
    w = plan.work_host  # {q_start, q_len, q_pos0, blk_begin, blk_count, q_pair, kv_head, n0|n1<<16}
    n0, n1 = plan.tiles_q0, plan.tiles_q1
    # GQA-4: 32 tokens per query tile, two tiles per item -> 1 pair for req 0, 9 for req 1
    assert plan.n_work == (1 + 9) * 8
    # L2 order: heaviest request first (req 1), grouped by kv head, longest pair first
    assert w[0, 0] == 32 and w[0, 6] == 0 and (n0[0], n1[0]) == (4, 4)
    for h in range(8):
        sel = (w[:, 0] == 32) & (w[:, 6] == h)
        tot = list(n0[sel] + n1[sel])
        assert tot == sorted(tot, reverse=True)
    r0 = (w[:, 0] == 0)  # request 0 starts at query row 0: one tile, Q1 empty
    assert set(n0[r0]) == {9} and set(n1[r0]) == {0}  # 1056 slots -> 9 key tiles
    assert set(map(tuple, w[r0, :5])) == {(0, 32, 1024, 0, 66)}
    r1 = (w[:, 0] == 32)
    # causal: query tile t covers tokens [32t, 32t+32) -> needs key tile (32t+31)//128;
    # the last pair (tokens 512..543) has an empty Q1
    got = sorted(set(zip(w[r1, 5], n0[r1], n1[r1])))
    need = lambda t: (32 * t + 31) // 128 + 1 if 32 * t < 544 else 0
    assert got == [(p, need(2 * p), need(2 * p + 1)) for p in range(9)]
    assert np.all(np.bincount(w[r1, 6]) == 9)
    # half flags: Q tile t's last key slot 32t+31 lies in the first 64 of its last KV tile
    for p, h0, h1 in zip(w[r1, 5], plan.half_q0[r1], plan.half_q1[r1]):
        assert h0 == ((64 * p + 31) % 128 < 64)
        assert h1 == (((64 * p + 63) % 128 < 64) if 64 * p + 32 < 544 else False)


def test_layered_swap_api_accounting_mode():
    """flush_layered / fence_layer / drain on an accounting pool (no device memory):
    batches are accounted like rcb_pool_flush, arguments are validated."""
    import pytest

    from paper_2404_12457_b200.pool import PoolError, accounting_pool

    pool = accounting_pool(32, 16, 16)
    pool.node_alloc_gpu(1, 40)  # 3 blocks
    pool.node_swap_out([1])
    pool.flush_layered(1)  # pending D2H: issued (accounted) as a normal batch
    assert pool.stats()["d2h_bytes"] == 3 * pool.block_bytes
    pool.node_swap_in([1])
    pool.flush_layered(4)  # layers_per_group larger than n_layers is clamped
    assert pool.stats()["h2d_bytes"] == 3 * pool.block_bytes
    pool.fence_layer(0, None)
    pool.drain()
    with pytest.raises(PoolError):
        pool.flush_layered(0)
    with pytest.raises(PoolError):
        pool.fence_layer(1, None)  # the accounting pool has one layer
    pool.close()


def test_attn_plan_split_only_flag():
    """Plans whose items are all lone query tiles select the split-only kernel variant."""
    import numpy as np

    # the host-only part of kernels.AttnPlan: the planner through the C-ABI
    def work_flags(reqs, g=4):
        meta, valid, pos = [], [], []
        q_start = 0
        for q_len, q_pos0 in reqs:
            n = -(-(q_pos0 + q_len) // 64)
            meta += [q_start, q_len, q_pos0, len(valid), n]
            for b in range(n):
                valid.append(min(64, q_pos0 + q_len - 64 * b))
                pos.append(64 * b)
            q_start += q_len
        requests = reqs
        cap = 4096
        work = np.zeros(cap * 8, dtype=np.int32)
        n = np.zeros(1, dtype=np.int32)
        lib = _lib.load()
        assert lib.rcb_attn_plan(np.asarray(meta, np.int32).ctypes.data_as(_lib._p32), len(requests),
                                 np.asarray(valid, np.int32).ctypes.data_as(_lib._p32),
                                 np.asarray(pos, np.int32).ctypes.data_as(_lib._p32), 64, 8 * g, 8,
                                 work.ctypes.data_as(_lib._p32), cap,
                                 n.ctypes.data_as(_lib._p32)) == 0
        tiles_q1 = (work[: n[0] * 8].reshape(-1, 8)[:, 7].view(np.uint32) >> 16) & 0x7FFF
        return 0 if tiles_q1.any() else _lib.RCB_WORK_SPLIT_ONLY

    assert work_flags([(1, 4096)] * 8) == _lib.RCB_WORK_SPLIT_ONLY      # decode
    assert work_flags([(32, 1024)] * 8) == _lib.RCB_WORK_SPLIT_ONLY     # full hits, 32-token prompt
    assert work_flags([(1056, 0)] * 2) == 0                              # misses: tile pairs
