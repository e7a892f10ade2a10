"""Layer-pipelined swap-in vs the serial swap-in + prefill.

    python tools/layered_swap.py [shape] [--no-cells] [--engine [--workload W] [--requests N]]

Part 1 (cells): one generation of k documents where `h` cached documents sit in
the pinned host tier (the knowledge tree's host hits, load_to_gpu tree.py:296-318)
and k - h are misses, plus a 32-token prompt. Per cell, CUDA-event time of
  * copy     : the swap-in alone (H2D of h x 512 tokens of KV),
  * compute  : the prefill alone with the cached pages already resident,
  * serial   : swap-in then prefill (what ragsim charges: transfer + T(a,b),
               simulator.py:505-510),
  * layered  : the swap-in issued per group of layers, layer l's attention waiting
               only for its group (BlockPool.flush_layered / fence_layer),
for several layers-per-group. Random-init weights of the shape; cuBLAS GEMMs and
our kernels.

Part 2 (--engine): TimedEngine on the llama2-7b-top5-qpool workload (configs[2]: GPU +
host tier under memory pressure, repeated questions so the host tier serves hits) with the swap-in modeled (ragsim's serial
transfer charge), executed serially, and executed layer-pipelined: p50/mean TTFT.

Writes $OUT_DIR (default profiles/)/<shape>_layered_swap.json.
"""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_12457_b200 import _lib, kernels  # noqa: E402
from paper_2404_12457_b200.model import DIMS, PrefillModel, init_weights, suffix_slots  # noqa: E402
from paper_2404_12457_b200.pool import BlockPool  # noqa: E402

DOC = 512
PROMPT = 32
BT = 64


def cells(shape: str, k: int, reps: int = 5):
    dims = DIMS[shape]
    s = dims.shape
    w = init_weights(dims, seed=0)
    nb_doc = DOC // BT
    ng = 2 * k * nb_doc + 16
    block_bytes = s.n_layers * 2 * s.n_kv_heads * BT * s.head_dim * 2
    kvbuf = torch.zeros((ng, block_bytes // 2), dtype=torch.bfloat16, device="cuda")
    pool = BlockPool(ng, k * nb_doc + 8, block_tokens=BT, n_layers=s.n_layers,
                     n_kv_heads=s.n_kv_heads, head_dim=s.head_dim, swap_mode=_lib.RCB_SWAP_DMA,
                     gpu_base=kvbuf.data_ptr())
    model = PrefillModel(dims, w, block_tokens=BT, num_pool_blocks=ng, pool_base=kvbuf.data_ptr())
    stream = torch.cuda.current_stream()
    # k host-resident document nodes with random KV
    for d in range(k):
        pool.node_alloc_gpu(1 + d, DOC)
        blocks = pool.node_blocks(1 + d)
        kvbuf[blocks] = torch.randn((len(blocks), block_bytes // 2), device="cuda").to(torch.bfloat16)
    torch.cuda.synchronize()
    pool.node_swap_out(list(range(1, k + 1)))
    pool.sync()
    tok_gen = torch.Generator().manual_seed(1)
    rows = []
    gen_key = [0]

    def one(h: int, mode: str, lpg: int = 4) -> float:
        hits = list(range(1, h + 1))
        misses = k - h
        seg = [DOC] * misses + [PROMPT]
        gk = gen_key[0]
        gen_key[0] += 1
        if mode != "compute":
            pool.node_swap_in(hits)
        else:  # resident: swap in outside the timed region
            pool.node_swap_in(hits)
            pool.fence_into(stream)
        pool.gen_reserve(gk, seg)
        blocks, valid = pool.block_table(hits, gk)
        alpha, beta = h * DOC, misses * DOC + PROMPT
        slots, pos = suffix_slots(blocks, valid, h * nb_doc, BT, alpha)
        plan = kernels.AttnPlan([(beta, alpha, blocks, valid)], block_tokens=BT,
                                n_q_heads=s.n_q_heads, n_kv_heads=s.n_kv_heads)
        tok = torch.randint(0, dims.vocab, (beta,), generator=tok_gen).cuda()
        posd = torch.tensor(pos, dtype=torch.int32, device="cuda")
        slotd = torch.tensor(slots, dtype=torch.int32, device="cuda")
        last = torch.tensor([beta - 1], device="cuda")
        torch.cuda.synchronize()
        pool.drain()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pool.wait_for(stream)
        fence = None
        if mode == "layered":
            pool.flush_layered(lpg)
            fence = lambda layer: pool.fence_layer(layer, stream)  # noqa: E731
        elif mode in ("serial", "copy"):
            pool.fence_into(stream)
        if mode != "copy":
            model.prefill(tok, posd, slotd, plan, last, layer_fence=fence)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        pool.gen_release(gk)
        for n in hits:  # host copy kept: the next swap-in of the same nodes is valid
            pool.node_free_gpu(n)
        return ms

    def med(h, mode, lpg=4):
        one(h, mode, lpg)  # warm-up
        return float(np.median([one(h, mode, lpg) for _ in range(reps)]))

    for h in range(1, k + 1):
        r = {"host_hit_docs": h, "miss_docs": k - h, "alpha": h * DOC,
             "beta": (k - h) * DOC + PROMPT,
             "h2d_bytes": h * DOC * s.kv_bytes_per_token,
             "copy_ms": round(med(h, "copy"), 3), "compute_ms": round(med(h, "compute"), 3),
             "serial_ms": round(med(h, "serial"), 3)}
        r["h2d_gbs"] = round(r["h2d_bytes"] / (r["copy_ms"] / 1e3) / 1e9, 2)
        r["layered_ms"] = {str(g): round(med(h, "layered", g), 3) for g in (1, 2, 4, 8)}
        best = min(r["layered_ms"].values())
        r["bound_ms"] = round(max(r["copy_ms"], r["compute_ms"]), 3)
        r["speedup_vs_serial"] = round(r["serial_ms"] / best, 3)
        rows.append(r)
        print(json.dumps(r), flush=True)
    pool.close()
    return rows


def engine(name: str, n_req: int, rate: float):
    from paper_2404_12457_b200 import cache  # noqa: F401
    from paper_2404_12457_b200.profile import decode_ms_per_token, measure_profile
    from paper_2404_12457_b200.timed import ModelExecutor, run_timed
    from paper_2404_12457_b200.workloads import WORKLOADS, make_stream, pool_blocks
    from ragsim.config import RunConfig
    from ragsim.cost_model import save_profile_csv

    w = WORKLOADS[name]
    prof, info = measure_profile(w.shape, block_tokens=w.block_tokens, reps=3)
    dec = decode_ms_per_token(prof, w.k * int(w.doc_tokens_mean) + w.prompt_tokens)
    path = os.path.join("/tmp", f"{w.shape}_layered_profile.csv")
    save_profile_csv(prof, path)
    pcie = measure_pcie()
    stage_ms = measure_stage_ms(w)
    trace, sizes = make_stream(w, n_req, rate=rate)
    host = int(os.environ.get("HOST_TIER_TOKENS", 64_000))
    cfg = RunConfig(gpu_capacity_tokens=w.gpu_capacity_tokens, host_capacity_tokens=host,
                    k=w.k, profile_path=path, decode_ms_per_token=dec,
                    kv_bytes_per_token=float(w.model.kv_bytes_per_token),
                    pcie_bandwidth_bytes_per_ms=pcie * 1e6, stage_interval_ms=stage_ms,
                    seed=w.seed)
    ng = pool_blocks(w.gpu_capacity_tokens, w.block_tokens, sizes.values(), 8 * (w.k + 1))
    nh = pool_blocks(host, w.block_tokens, sizes.values(), 0)
    s = w.model
    pool = None
    ex = None
    out = {"workload": w.name, "requests": n_req, "rate_req_s": rate, "host_tier_tokens": host,
           "gpu_tier_tokens": w.gpu_capacity_tokens, "pcie_h2d_gbs": round(pcie, 2),
           "decode_ms_per_token": round(dec, 3), "stage_interval_ms": round(stage_ms, 4),
           "modes": {}}
    for mode in ("modeled", "serial", "layered"):
        t0 = time.time()
        pool = BlockPool(ng, nh, block_tokens=w.block_tokens, n_layers=s.n_layers,
                         n_kv_heads=s.n_kv_heads, head_dim=s.head_dim,
                         swap_mode=_lib.RCB_SWAP_DMA)
        if ex is None:
            ex = ModelExecutor(pool, w.shape, swap_in=mode)
        else:  # reuse the weights; rebind to the fresh pool
            ex = rebind(ex, pool, mode)
        rep, eng = run_timed(cfg, trace, sizes, pool=pool, executor=ex)
        pool.sync()
        a = rep.aggregates()
        st = pool.stats()
        # admissions with host-tier hits: transfer + prefill charged on the critical path
        hh = [t + p for _, mt, t, p in eng.critical if mt > 0]
        out["modes"][mode] = {"p50_ttft_ms": round(a["median_ttft_ms"], 3),
                              "mean_ttft_ms": round(a["mean_ttft_ms"], 3),
                              "doc_hit_rate": round(a["doc_hit_rate"], 4),
                              "swap_in_blocks": st["swap_in_blocks"],
                              "host_hit_admissions": len(hh),
                              "host_hit_admit_ms_mean": round(float(np.mean(hh)), 3) if hh else None,
                              "host_hit_admit_ms_p50": round(float(np.median(hh)), 3) if hh else None,
                              "swap_out_blocks": st["swap_out_blocks"],
                              "seconds": round(time.time() - t0, 1)}
        print(mode, json.dumps(out["modes"][mode]), flush=True)
        pool.close()
    return out


def rebind(ex, pool, mode):
    from paper_2404_12457_b200.timed import ModelExecutor

    new = ModelExecutor.__new__(ModelExecutor)
    new.__dict__.update(ex.__dict__)
    new.pool = pool
    new.swap_in = mode
    new.model = PrefillModel(ex.dims, ex.w, block_tokens=pool.block_tokens,
                             num_pool_blocks=pool.num_gpu_blocks, pool_base=pool.gpu_base)
    return new


def measure_stage_ms(w) -> float:
    """Measured retrieval stage interval: a 64-query staged scan of the corpus / stages."""
    from paper_2404_12457_b200 import synth

    corpus = synth.corpus_device(w.num_docs, seed=w.seed)
    q = torch.randint(-100, 100, (64, synth.EMB_DIM), device="cuda").to(torch.bfloat16)
    ws = kernels.RetrievalWorkspace(w.num_docs, 64, w.k, w.n_stages)
    kernels.retrieval_topk(corpus, q, w.k, w.n_stages, workspace=ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        kernels.retrieval_topk(corpus, q, w.k, w.n_stages, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10 / w.n_stages


def measure_pcie() -> float:
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    shape = args[0] if args else "llama2-7b"
    k = int(sys.argv[sys.argv.index("--k") + 1]) if "--k" in sys.argv else 5
    out = {"shape": shape, "k": k, "doc_tokens": DOC, "prompt_tokens": PROMPT,
           "block_tokens": BT, "timing": "CUDA events, median of 5, swap-outs drained first",
           "cells": [] if "--no-cells" in sys.argv else cells(shape, k)}
    torch.cuda.empty_cache()
    if "--engine" in sys.argv:
        n_req = int(sys.argv[sys.argv.index("--requests") + 1]) if "--requests" in sys.argv else 300
        rate = float(sys.argv[sys.argv.index("--rate") + 1]) if "--rate" in sys.argv else 1.0
        name = (sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv
                else "llama2-7b-top5-qpool")
        out["engine"] = engine(name, n_req, rate)
    out_dir = os.environ.get("OUT_DIR", os.path.join(ROOT, "profiles"))
    os.makedirs(out_dir, exist_ok=True)
    json.dump(out, open(os.path.join(out_dir, f"{shape}_layered_swap.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
