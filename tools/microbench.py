"""Per-kernel microbenchmarks on one GPU (CUDA events, warm, inputs > L2 or flushed).

    python tools/microbench.py [pcie|copy|swap|retrieval|attn|all] [--ncu]

Prints one JSON object per measurement.  --ncu runs each kernel only a few
times (for `ncu --set full` captures; numbers printed under ncu are not
measurements).
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_12457_b200 import _lib, kernels, synth  # noqa: E402
from paper_2404_12457_b200.pool import BlockPool  # noqa: E402

NCU = "--ncu" in sys.argv
REPS = 2 if NCU else 20
L2_FLUSH = None


def flush_l2():
    global L2_FLUSH
    if L2_FLUSH is None:
        L2_FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L2_FLUSH.zero_()


def timed(fn, reps=REPS, flush=True):
    ts = []
    for _ in range(2 if not NCU else 0):
        fn()
    for _ in range(reps):
        if flush:
            flush_l2()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(np.min(ts))


def emit(**kw):
    print(json.dumps(kw), flush=True)


def peaks():
    p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    return p["hbm_gbs"], p["bf16_tflops"]


def bench_pcie():
    n = 1 << 30
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2d, _ = timed(lambda: dev.copy_(host, non_blocking=True), reps=5, flush=False)
    d2h, _ = timed(lambda: host.copy_(dev, non_blocking=True), reps=5, flush=False)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    host2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    dev2 = torch.empty(n, dtype=torch.uint8, device="cuda")

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            dev.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2):
            host2.copy_(dev2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    duplex, _ = timed(both, reps=5, flush=False)
    emit(kind="pcie_pinned_memcpy", bytes=n, h2d_gbs=n / h2d / 1e6, d2h_gbs=n / d2h / 1e6,
         duplex_gbs=2 * n / duplex / 1e6)
    return n / h2d / 1e6, n / d2h / 1e6


def bench_copy():
    hbm, _ = peaks()
    for block_bytes, n_pairs in ((8 << 20, 128), (2 << 20, 512), (32768, 16384)):
        nb = n_pairs * 2
        src = torch.empty(nb * block_bytes, dtype=torch.uint8, device="cuda")
        dst = torch.empty_like(src)
        rng = np.random.default_rng(0)
        pairs = torch.tensor(np.stack([rng.permutation(nb)[:n_pairs], rng.permutation(nb)[:n_pairs]], 1),
                             dtype=torch.int32, device="cuda")
        med, best = timed(lambda: kernels.block_copy(src.data_ptr(), dst.data_ptr(), block_bytes, pairs))
        moved = 2 * n_pairs * block_bytes
        emit(kind="block_gather_hbm", block_bytes=block_bytes, pairs=n_pairs, ms=med,
             gbs=moved / med / 1e6, frac_hbm=moved / med / 1e6 / hbm)
        del src, dst


def bench_swap():
    """Pool swap paths, Mistral-7B geometry, 64-token (8 MiB) blocks, 96 nodes x 8 blocks."""
    import time

    geom = dict(block_tokens=64, n_layers=32, n_kv_heads=8, head_dim=128)
    for mode, name in ((0, "staged"), (1, "zerocopy"), (2, "dma")):
        pool = BlockPool(1024, 1024, swap_mode=mode, **geom)
        keys = list(range(96))
        for k in keys:
            pool.node_alloc_gpu(k, 512)
        pool.sync()
        ts_out, ts_in = [], []
        for _ in range(2 if NCU else 5):
            t0 = time.perf_counter()
            pool.node_swap_out(keys)  # GPU -> host, GPU blocks freed
            pool.sync()
            t1 = time.perf_counter()
            pool.node_swap_in(keys)  # host -> GPU, host copy kept
            pool.sync()
            t2 = time.perf_counter()
            for k in keys:
                pool.node_free_host(k)
            ts_out.append(t1 - t0)
            ts_in.append(t2 - t1)
        nbytes = len(keys) * 8 * pool.block_bytes
        emit(kind="pool_swap", mode=name, block_bytes=pool.block_bytes, bytes=nbytes,
             d2h_gbs=nbytes / float(np.median(ts_out)) / 1e9,
             h2d_gbs=nbytes / float(np.median(ts_in)) / 1e9)
        pool.close()


def bench_retrieval():
    hbm, _ = peaks()
    n = 100_000
    corpus = synth.corpus_device(n, seed=0)
    # shard-scale comparison: a 10M corpus over 8 ranks is a 1.25M-row shard per rank, and the
    # ranks' all-gathered queries come to 8 x 32 = 256 per step: one pass of 256 (a 4-CTA
    # cluster per range, corpus stages multicast) against four passes of 64
    shard = synth.corpus_device(1_250_000, seed=0)
    qb = torch.randint(-100, 100, (256, synth.EMB_DIM), device="cuda").to(torch.bfloat16)
    ws256 = kernels.RetrievalWorkspace(shard.shape[0], 256, 2, 4)
    ws64 = kernels.RetrievalWorkspace(shard.shape[0], 64, 2, 4)
    ws128 = kernels.RetrievalWorkspace(shard.shape[0], 128, 2, 4)
    one, _ = timed(lambda: kernels.retrieval_topk(shard, qb, 2, 4, workspace=ws256))
    two, _ = timed(lambda: [kernels.retrieval_topk(shard, qb[i:i + 128], 2, 4, workspace=ws128)
                            for i in range(0, 256, 128)])
    four, _ = timed(lambda: [kernels.retrieval_topk(shard, qb[i:i + 64], 2, 4, workspace=ws64)
                             for i in range(0, 256, 64)])
    sb = shard.shape[0] * synth.EMB_DIM * 2
    emit(kind="retrieval_shard_256q", rows=shard.shape[0], queries=256, one_pass_ms=one,
         two_passes_of_128_ms=two, four_passes_of_64_ms=four, one_pass_gbs=sb / one / 1e6,
         one_pass_frac_hbm=sb / one / 1e6 / hbm)
    del shard, ws256, ws64, ws128
    for b in (256, 128, 64, 32, 16, 1):
        q = torch.randint(-100, 100, (b, synth.EMB_DIM), device="cuda").to(torch.bfloat16)
        ws = kernels.RetrievalWorkspace(n, b, 2, 4)
        ids = torch.empty((b, 4, 2), dtype=torch.int64, device="cuda")
        sc = torch.empty((b, 4, 2), dtype=torch.float32, device="cuda")
        med, best = timed(lambda: kernels.retrieval_topk(corpus, q, 2, 4, workspace=ws, ids_out=ids,
                                                         scores_out=sc))
        emit(kind="retrieval_topk", rows=n, dim=synth.EMB_DIM, queries=b, ms=med,
             gbs=n * synth.EMB_DIM * 2 / med / 1e6, frac_hbm=n * synth.EMB_DIM * 2 / med / 1e6 / hbm)
        if NCU:
            continue
        # device-side time without host launch gaps: 20 calls captured in a CUDA graph
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            kernels.retrieval_topk(corpus, q, 2, 4, workspace=ws, ids_out=ids, scores_out=sc)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    kernels.retrieval_topk(corpus, q, 2, 4, workspace=ws, ids_out=ids,
                                           scores_out=sc)
        torch.cuda.synchronize()
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        gms = e0.elapsed_time(e1) / 20
        # host cost of one call (no sync): wall time of 200 back-to-back calls
        import time as _t
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        for _ in range(200):
            kernels.retrieval_topk(corpus, q, 2, 4, workspace=ws, ids_out=ids, scores_out=sc)
        host_us = (_t.perf_counter() - t0) / 200 * 1e6
        torch.cuda.synchronize()
        emit(kind="retrieval_topk_graph", rows=n, queries=b, ms=gms,
             gbs=n * synth.EMB_DIM * 2 / gms / 1e6, frac_hbm=n * synth.EMB_DIM * 2 / gms / 1e6 / hbm,
             host_us_per_call=round(host_us, 1))


def bench_attn():
    _, tc = peaks()
    cases = [
        ("mistral hit a1024 b32 x64", 32, 8, 64, [(1024, 32)] * 64),
        ("mistral miss a0 b1056 x16", 32, 8, 64, [(0, 1056)] * 16),
        ("mistral mixed step", 32, 8, 64, [(0, 1056)] * 26 + [(512, 544)] * 26 + [(1024, 32)] * 12),
        ("llama2 miss a0 b544 x16", 32, 32, 64, [(0, 544)] * 16),
        ("mistral long a4096 b256 x32", 32, 8, 64, [(4096, 256)] * 32),
        # a decode step: one new token per request over its cached context (HBM-bound)
        ("mistral decode a1056 b1 x64", 32, 8, 64, [(1056, 1)] * 64),
        ("mistral decode a4096 b1 x64", 32, 8, 64, [(4096, 1)] * 64),
        # one request (the TTFT engine's single-server decode step / cached-prefix prompt):
        # 8 items, split-KV across the SMs
        ("mistral decode a1056 b1 x1", 32, 8, 64, [(1056, 1)]),
        ("mistral hit a1024 b32 x1", 32, 8, 64, [(1024, 32)]),
    ]
    only = os.environ.get("MB_CASE")
    for name, hq, hkv, bt, reqs in cases:
        if only and only not in name:
            continue
        hd, L = 128, 2
        total_slots = sum(-(-(a + b) // bt) for a, b in reqs)
        nb = total_slots + 8
        pool = (torch.randn((nb, L, 2, hkv, bt, hd), device="cuda") * 0.5).to(torch.bfloat16)
        perm = np.random.default_rng(0).permutation(nb)
        requests, pos = [], 0
        for a, b in reqs:
            n = -(-(a + b) // bt)
            blocks = [int(x) for x in perm[pos:pos + n]]
            pos += n
            valid = [bt] * (n - 1) + [a + b - (n - 1) * bt]
            requests.append((b, a, blocks, valid))
        T = sum(b for _, b in reqs)
        q = (torch.randn((T, hq, hd), device="cuda")).to(torch.bfloat16)
        o = torch.empty_like(q)
        plan = kernels.AttnPlan(requests, block_tokens=bt, n_q_heads=hq, n_kv_heads=hkv)
        fn = lambda: kernels.prefix_prefill(q, o, plan, pool.data_ptr(), nb, block_tokens=bt,
                                            n_layers=L, n_kv_heads=hkv, head_dim=hd, layer=1)
        med, best = timed(fn)
        flops = sum(4.0 * hq * hd * (a * b + b * (b + 1) / 2) for a, b in reqs)
        kv_bytes = sum((a + b) * 2 * hkv * hd * 2 for a, b in reqs)
        emit(kind="prefix_prefill", case=name, ms=med, tflops=flops / med / 1e9,
             frac_tc=flops / med / 1e9 / tc, kv_gbs=kv_bytes / med / 1e6, work_items=plan.n_work,
             kv_tiles=plan.kv_tiles)
        # fused Q-RoPE: raw Q columns of a QKV row, rotated in shared memory
        qkv = torch.randn((T, (hq + 2 * hkv) * hd), device="cuda").to(torch.bfloat16)
        rope = kernels.rope_table(plan.max_pos + 1, hd, 1e6)
        fn = lambda: kernels.prefix_prefill(qkv[:, : hq * hd], o, plan, pool.data_ptr(), nb,
                                            block_tokens=bt, n_layers=L, n_kv_heads=hkv,
                                            head_dim=hd, layer=1, rope=rope, n_q_heads=hq)
        med, best = timed(fn)
        emit(kind="prefix_prefill_rope", case=name, ms=med, tflops=flops / med / 1e9,
             frac_tc=flops / med / 1e9 / tc)
        fn = lambda: kernels.prefix_prefill(q, o, plan, pool.data_ptr(), nb,
                                            block_tokens=bt, n_layers=L, n_kv_heads=hkv,
                                            head_dim=hd, layer=1, rope=rope, n_q_heads=hq)
        med, best = timed(fn)
        emit(kind="prefix_prefill_rope_contig_q", case=name, ms=med, tflops=flops / med / 1e9)
        pos_t = torch.cat([a + torch.arange(b) for a, b in reqs]).to(torch.int32).cuda()
        slots = torch.arange(T, dtype=torch.int32, device="cuda")
        x = qkv
        k = x[:, hq * hd:(hq + hkv) * hd]
        v = x[:, (hq + hkv) * hd:]
        qr = torch.empty((T, hq, hd), dtype=torch.bfloat16, device="cuda")
        for mode, qq, qo, tab in (("qkv", x[:, : hq * hd], qr, None),
                                  ("qkv_table", x[:, : hq * hd], qr, rope),
                                  ("kv_only", None, None, None),
                                  ("kv_only_table", None, None, rope)):
            mp = int(pos_t.max()) + 1  # outside the timed call (a device sync)
            fn = lambda: kernels.kv_write_rope(qq, k, v, qo, pos_t, slots, pool.data_ptr(),
                                               block_tokens=bt, n_layers=L, n_kv_heads=hkv,
                                               head_dim=hd, layer=1, rope_theta=1e6, n_q_heads=hq,
                                               rope=tab, max_pos=mp)
            med, best = timed(fn)
            nbytes = T * hd * 2 * (2 * hkv * 2 + (2 * hq if qq is not None else 0))
            emit(kind="kv_write_rope", mode=mode, case=name, ms=med, gbs=nbytes / med / 1e6)
        del pool


if __name__ == "__main__":
    which = [a for a in sys.argv[1:] if not a.startswith("--")] or ["all"]
    torch.cuda.set_device(0)
    _lib.load()
    table = {"pcie": bench_pcie, "copy": bench_copy, "swap": bench_swap,
             "retrieval": bench_retrieval, "attn": bench_attn}
    for name, fn in table.items():
        if "all" in which or name in which:
            fn()
