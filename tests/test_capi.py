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
    w = plan.work_host  # {q_start, q_len, q_pos0, blk_begin, blk_count, q_tile, kv_head, n}
    # GQA-4: 32 tokens per query tile -> 1 tile for req 0, 17 for req 1, x 8 kv heads
    assert plan.n_work == (1 + 17) * 8
    # L2 order: heaviest request first (req 1: 17 q-tiles), grouped by kv head,
    # longest q-tile first within a group
    assert w[0, 0] == 32 and w[0, 6] == 0 and w[0, 7] == 5
    for h in range(8):
        grp = w[(w[:, 0] == 32) & (w[:, 6] == h)]
        assert list(grp[:, 7]) == sorted(grp[:, 7], reverse=True)
    r0 = w[w[:, 0] == 0]  # request 0 starts at query row 0
    assert set(r0[:, 7]) == {9}  # 1056 slots -> 9 key tiles
    assert set(map(tuple, r0[:, :5])) == {(0, 32, 1024, 0, 66)}
    r1 = w[w[:, 0] == 32]
    # causal: query tile t covers tokens [32t, 32t+32) -> needs key tile (32t+31)//128
    assert sorted(set(zip(r1[:, 5], r1[:, 7]))) == [(t, (32 * t + 31) // 128 + 1) for t in range(17)]
    assert np.all(np.bincount(r1[:, 6]) == 17)
