"""Re-run the reference's policy / reordering / DSP acceptance trends (C5, C6, C7:
pkg/tests/test_acceptance.py:252-361; the C5 sweep is pkg/scripts/policy_sweep.py:31) on
B200-measured costs instead of ragsim's synthetic ones.

The recipes (desk MMLU corpus, question pool with drift, capacities, seeds, thresholds) are
the reference's.  Only the cost inputs change:
  * prefill T(alpha, beta): profiles/llama2-7b_b200_profile.csv (the desk recipe's
    kv_bytes_per_token = 0.5 MiB is LLaMA2-7B's KV size), through RunConfig.profile_path
  * decode: the measured one-token step (profiles/llama2-7b_b200_profile.json) instead of
    the 20 ms constant (config.py:52)
  * host<->GPU: the measured pinned-copy GB/s instead of 16 GiB/s (cost_model.py:74-75)
  * C7 twice: the reference's 50 ms stage interval (a CPU vector search)
    and the B200 retrieval kernel's measured per-stage time.
Writes profiles/r2_acceptance_b200.json.  CPU only (ragsim's engine, unmodified).

    python tools/acceptance_b200.py [--quick]
"""

import dataclasses
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_12457_b200._ragsim import import_ragsim  # noqa: E402

import_ragsim()
from ragsim.config import RunConfig  # noqa: E402
from ragsim.policies import POLICY_NAMES  # noqa: E402
from ragsim.simulator import measure_throughput, run, scale_trace  # noqa: E402
from ragsim.workload import PRESETS, TraceSpec, generate_corpus, generate_trace  # noqa: E402

MIB = 1024.0 * 1024.0
CORPUS = dataclasses.replace(PRESETS["mmlu"], num_docs=1500)
TRACE = dict(query_pool=400, query_zipf_s=1.1, drift_interval_s=300.0, drift_fraction=0.3)
HIT_EPS, TTFT_EPS_MS = 0.005, 0.5  # the reference's statistical-tie tolerances

# the reference's desk cost model (pkg/tests/test_acceptance.py:37-43)
SYNTHETIC = dict(gpu_capacity_tokens=10240, profile_base_ms=20.0, profile_per_token_ms=0.015,
                 profile_attention_ms=1e-5, kv_bytes_per_token=0.5 * MIB)


def b200_costs(pcie_gbs: float = 55.0) -> dict:
    info = json.load(open(os.path.join(ROOT, "profiles", "llama2-7b_b200_profile.json")))
    return dict(gpu_capacity_tokens=10240, kv_bytes_per_token=0.5 * MIB,
                profile_path=os.path.join(ROOT, "profiles", "llama2-7b_b200_profile.csv"),
                decode_ms_per_token=float(info["decode_ms_per_token"]["1056"]),
                pcie_bandwidth_bytes_per_ms=pcie_gbs * 1e9 / 1e3)


def trace_for(seed, duration_s, rate, pool=400):
    rng = np.random.default_rng(np.random.SeedSequence([seed]))
    corpus = generate_corpus(CORPUS, rng)
    spec = TraceSpec(duration_s=duration_s, arrival_rate=rate, seed=seed,
                     **{**TRACE, "query_pool": pool})
    return generate_trace(corpus, spec, rng), corpus.size_map()


def c5(costs, seeds=(0, 1, 2), caps=(12288, 20480, 32768, 49152, 73728)):
    cells = []
    for seed in seeds:
        trace, sizes = trace_for(seed, 3600.0, 0.8)
        for cap in caps:
            cell = {}
            for policy in POLICY_NAMES:
                cfg = RunConfig(host_capacity_tokens=cap, policy=policy, seed=seed, **costs)
                a = run(cfg, trace, sizes).aggregates()
                cell[policy] = (a["doc_hit_rate"], a["mean_ttft_ms"])
            cells.append({"seed": seed, "host_capacity_tokens": cap, **cell})
    base = ("gdsf", "lru", "lfu")
    hit_wins = sum(all(c["pgdsf"][0] >= c[p][0] - HIT_EPS for p in base) for c in cells)
    ttft_wins = sum(all(c["pgdsf"][1] <= c[p][1] + TTFT_EPS_MS for p in base) for c in cells)
    mean_hit = {p: float(np.mean([c[p][0] for c in cells])) for p in POLICY_NAMES}
    mean_ttft = {p: float(np.mean([c[p][1] for c in cells])) for p in POLICY_NAMES}
    need = int(np.ceil(0.9 * len(cells)))
    passed = (hit_wins >= need and ttft_wins >= need
              and all(mean_hit["pgdsf"] > mean_hit[p] for p in base)
              and mean_ttft["pgdsf"] < mean_ttft["lru"] and mean_ttft["pgdsf"] < mean_ttft["lfu"]
              and mean_ttft["pgdsf"] <= mean_ttft["gdsf"] + 0.05)
    return {"pass": bool(passed), "hit_cells": f"{hit_wins}/{len(cells)}",
            "ttft_cells": f"{ttft_wins}/{len(cells)}",
            "mean_hit": {k: round(v, 4) for k, v in mean_hit.items()},
            "mean_ttft_ms": {k: round(v, 3) for k, v in mean_ttft.items()}, "cells": cells}


def c6(costs, max_rate):
    trace, sizes = trace_for(0, 400.0, 1.0)
    fifo = RunConfig(host_capacity_tokens=20480, reorder=False, seed=0, **costs)
    sat = measure_throughput(fifo, trace, sizes, slo_multiplier=5.0, min_rate=0.5,
                             max_rate=max_rate, iterations=8)
    base_rate = len(trace) / (max(r.arrival_ms for r in trace) / 1000.0)
    over = scale_trace(trace, base_rate / (1.2 * sat))
    t_fifo = run(fifo, over, sizes).aggregates()["mean_ttft_ms"]
    t_re = run(dataclasses.replace(fifo, reorder=True, reorder_window=64), over, sizes) \
        .aggregates()["mean_ttft_ms"]
    red = 1.0 - t_re / t_fifo
    return {"pass": bool(red >= 0.10), "saturation_req_s": round(sat, 3),
            "mean_ttft_fifo_ms": round(t_fifo, 2), "mean_ttft_reorder_ms": round(t_re, 2),
            "reduction": round(red, 4)}


def c7(costs, stage_ms):
    trace, sizes = trace_for(0, 500.0, 0.25, pool=300)
    base = dict(host_capacity_tokens=32768, stage_count=4, stage_interval_ms=stage_ms,
                convergence_stage=2, prefill_chunk_ms=25.0, seed=0, **costs)
    off = run(RunConfig(dsp=False, **base), trace, sizes).aggregates()
    on = run(RunConfig(dsp=True, **base), trace, sizes).aggregates()
    ratio = off["mean_non_overlap_ms"] / max(1e-12, on["mean_non_overlap_ms"])
    return {"pass": bool(ratio >= 1.2 and on["mean_ttft_ms"] < off["mean_ttft_ms"]),
            "stage_interval_ms": stage_ms,
            "non_overlap_ms": [round(off["mean_non_overlap_ms"], 3),
                               round(on["mean_non_overlap_ms"], 3)],
            "ratio": round(ratio, 3),
            "mean_ttft_ms": [round(off["mean_ttft_ms"], 3), round(on["mean_ttft_ms"], 3)]}


def main():
    quick = "--quick" in sys.argv
    seeds = (0,) if quick else (0, 1, 2)
    bench = os.path.join(ROOT, "profiles", "r2_retrieval_stage_ms.json")
    stage_b200 = json.load(open(bench))["stage_ms"] if os.path.exists(bench) else 0.08
    out = {"recipe": "pkg/tests/test_acceptance.py desk MMLU (C5 :252-300, C6 :303-331, "
                      "C7 :334-361), thresholds unchanged",
           "b200_costs": {k: v for k, v in b200_costs().items() if k != "profile_path"},
           "b200_profile": "profiles/llama2-7b_b200_profile.csv"}
    for name, costs, max_rate in (("synthetic", SYNTHETIC, 16.0), ("b200", b200_costs(), 400.0)):
        t0 = time.time()
        res = {"c5": c5(costs, seeds=seeds), "c6": c6(costs, max_rate),
               "c7": c7(costs, 50.0)}
        if name == "b200":
            res["c7_b200_retrieval"] = c7(costs, stage_b200)
        res["seconds"] = round(time.time() - t0, 1)
        out[name] = res
        print(name, json.dumps({k: ({kk: vv for kk, vv in v.items() if kk != "cells"}
                                    if isinstance(v, dict) else v) for k, v in res.items()}),
              flush=True)
    path = os.path.join(os.environ.get("OUT_DIR", os.path.join(ROOT, "profiles")),
                        "r2_acceptance_b200.json")
    with open(path, "w") as fp:
        json.dump(out, fp, indent=1)


if __name__ == "__main__":
    main()
