"""Hardware-in-the-loop TTFT vs the measured-profile TTFT.

    python tools/timed_ttft.py [workload] [--requests N] [--rate R]

For each GPU tier, the reference engine runs the same trace twice. First on the
measured T(alpha, beta) grid (profile.py, interpolated). Then with TimedEngine, where
every admitted generation's prefill is executed on the GPU: a random-init model of the
workload's shape, cuBLAS GEMMs and our kernels on its real block table in a device pool
of the tier's size. Its CUDA-event time advances the clock. Writes
profiles/<workload>_timed_ttft.json ($OUT_DIR overrides the directory).
"""

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_12457_b200 import cache, kernels, synth  # noqa: E402
from paper_2404_12457_b200.pool import BlockPool, accounting_pool  # noqa: E402
from paper_2404_12457_b200.profile import decode_ms_per_token, measure_profile  # noqa: E402
from paper_2404_12457_b200.timed import ModelExecutor, run_timed  # noqa: E402
from paper_2404_12457_b200.workloads import WORKLOADS, make_stream, pool_blocks  # noqa: E402
from ragsim.config import RunConfig  # noqa: E402
from ragsim.cost_model import save_profile_csv  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name = args[0] if args else "mistral7b-100k-qpool"
    n_req = int(sys.argv[sys.argv.index("--requests") + 1]) if "--requests" in sys.argv else 400
    rate = float(sys.argv[sys.argv.index("--rate") + 1]) if "--rate" in sys.argv else 2.0
    w = WORKLOADS[name]
    t0 = time.time()
    prof, info = measure_profile(w.shape, block_tokens=w.block_tokens, reps=3)
    dec = decode_ms_per_token(prof, w.k * int(w.doc_tokens_mean) + w.prompt_tokens)
    t_prof = time.time() - t0
    # measured retrieval stage interval (64-query batch scan of the corpus / stages)
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
    stage_ms = e0.elapsed_time(e1) / 10 / w.n_stages
    del corpus
    path = os.path.join("/tmp", f"{w.shape}_timed_profile.csv")
    save_profile_csv(prof, path)
    trace, sizes = make_stream(w, n_req, rate=rate)
    floor = w.k * int(w.doc_tokens_mean) + w.prompt_tokens + 64
    tiers = sorted({max(floor, t) for t in (2200, 55_000)})
    rows = []
    for cap in tiers:
        cfg = RunConfig(gpu_capacity_tokens=cap, host_capacity_tokens=w.host_capacity_tokens,
                        k=w.k, profile_path=path, decode_ms_per_token=dec,
                        stage_interval_ms=stage_ms,
                        kv_bytes_per_token=float(w.model.kv_bytes_per_token), seed=w.seed)
        ng = pool_blocks(cap, w.block_tokens, sizes.values(), 8 * (w.k + 1))
        nh = pool_blocks(w.host_capacity_tokens, w.block_tokens, sizes.values(), 0) or 1
        t1 = time.time()
        prof_rep, _ = cache.run_tiered(cfg, trace, sizes, pool=accounting_pool(ng, nh, w.block_tokens))
        s = w.model
        pool = BlockPool(ng, nh, block_tokens=w.block_tokens, n_layers=s.n_layers,
                         n_kv_heads=s.n_kv_heads, head_dim=s.head_dim)
        ex = ModelExecutor(pool, w.shape)
        timed_rep, engine = run_timed(cfg, trace, sizes, pool=pool, executor=ex)
        pool.sync()
        torch.cuda.synchronize()
        a, b = prof_rep.aggregates(), timed_rep.aggregates()
        ratio = [m / p for _, _, _, p, m in engine.measured if p > 0]
        rows.append({"gpu_tier_tokens": cap,
                     "profile": {"doc_hit_rate": round(a["doc_hit_rate"], 4),
                                 "p50_ttft_ms": round(a["median_ttft_ms"], 3),
                                 "mean_ttft_ms": round(a["mean_ttft_ms"], 3)},
                     "timed": {"doc_hit_rate": round(b["doc_hit_rate"], 4),
                               "p50_ttft_ms": round(b["median_ttft_ms"], 3),
                               "mean_ttft_ms": round(b["mean_ttft_ms"], 3)},
                     "prefills_executed": len(engine.measured),
                     "measured_over_profile_median": round(sorted(ratio)[len(ratio) // 2], 3),
                     "pool_swap_out_blocks": pool.stats()["swap_out_blocks"],
                     "seconds": round(time.time() - t1, 1)})
        pool.close()
        del ex
        torch.cuda.empty_cache()
        print(json.dumps(rows[-1]), flush=True)
    out = {"workload": name, "shape": w.shape, "requests": n_req, "rate_req_s": rate,
           "decode_ms_per_token": round(dec, 3), "stage_interval_ms": round(stage_ms, 4),
           "profile": info,
           "profile_seconds": round(t_prof, 1), "tiers": rows}
    out_dir = os.environ.get("OUT_DIR", os.path.join(ROOT, "profiles"))  # gpurun: gpurun_out
    os.makedirs(out_dir, exist_ok=True)
    json.dump(out, open(os.path.join(out_dir, f"{name}_timed_ttft.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
