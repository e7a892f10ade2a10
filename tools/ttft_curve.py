"""Measured-profile loop: B200 T(alpha,beta) grid -> ragsim engine -> p50 TTFT vs hit rate.

    python tools/ttft_curve.py [workload] [--requests N] [--rate R]

Writes profiles/<shape>_b200_profile.csv (ragsim's format, cost_model.py:150-157)
and prints/saves the curve JSON (profiles/<workload>_ttft_curve.json).
"""

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_12457_b200 import kernels, synth  # noqa: E402
from paper_2404_12457_b200.profile import decode_ms_per_token, measure_profile  # noqa: E402
from paper_2404_12457_b200.retrieval import GpuStageProvider, synthetic_query_fn  # noqa: E402
from paper_2404_12457_b200.ttft import ttft_curve  # noqa: E402
from paper_2404_12457_b200.workloads import WORKLOADS  # noqa: E402
from ragsim.cost_model import save_profile_csv  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name = args[0] if args else "mistral7b-100k"
    n_req = int(sys.argv[sys.argv.index("--requests") + 1]) if "--requests" in sys.argv else 3000
    rate = float(sys.argv[sys.argv.index("--rate") + 1]) if "--rate" in sys.argv else 2.0
    w = WORKLOADS[name]
    t0 = time.time()
    prof, info = measure_profile(w.shape, block_tokens=w.block_tokens)
    t_prof = time.time() - t0
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    save_profile_csv(prof, os.path.join(os.environ.get("OUT_DIR", os.path.join(ROOT, "profiles")),
                                        f"{w.shape}_b200_profile.csv"))
    corpus = synth.corpus_device(w.num_docs, seed=w.seed)
    # measured per-stage scan time (64-query batch) -> stage interval
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

    def provider(trace, cfg):
        return GpuStageProvider(corpus, synthetic_query_fn(w.seed), k=w.k, n_stages=cfg.stage_count,
                                stage_interval_ms=stage_ms, trace=trace)

    if w.host_capacity_tokens:
        tiers = [w.gpu_capacity_tokens // 4, w.gpu_capacity_tokens // 2, w.gpu_capacity_tokens,
                 2 * w.gpu_capacity_tokens]
    else:
        tiers = [int(x * w.gpu_capacity_tokens) for x in (0.002, 0.01, 0.05, 0.2, 0.5, 1.0)]
    floor = w.k * int(w.doc_tokens_mean) + w.prompt_tokens + 64
    tiers = sorted({max(floor, t) for t in tiers})
    t1 = time.time()
    decode_ms = decode_ms_per_token(prof, w.k * int(w.doc_tokens_mean) + w.prompt_tokens)
    rows = ttft_curve(w, prof, gpu_tiers=tiers, host_tier=w.host_capacity_tokens,
                      n_requests=n_req, rate=rate, stage_provider_fn=provider,
                      decode_ms_per_token=decode_ms)
    out = {"workload": name, "shape": w.shape, "profile": info, "profile_seconds": round(t_prof, 1),
           "stage_interval_ms": round(stage_ms, 4), "decode_ms_per_token": round(decode_ms, 3),
           "rate_req_s": rate, "requests": n_req,
           "engine_seconds": round(time.time() - t1, 1),
           "profile_ms": {f"a{a}_b{b}": round(prof.times[i][j], 3)
                          for i, a in enumerate(prof.alpha_grid) for j, b in enumerate(prof.beta_grid)},
           "curve": rows}
    base = rows[0]["p50_ttft_ms"]
    for r in rows:
        r["p50_speedup_vs_smallest_tier"] = round(base / r["p50_ttft_ms"], 3)
    out_dir = os.environ.get("OUT_DIR", os.path.join(ROOT, "profiles"))  # gpurun: gpurun_out
    os.makedirs(out_dir, exist_ok=True)
    json.dump(out, open(os.path.join(out_dir, f"{name}_ttft_curve.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
