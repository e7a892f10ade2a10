"""p50 TTFT and hit rate vs cache size on B200 costs (the measured-profile loop).

Runs the reference's engine (decisions, queueing, DSP, virtual clock —
simulator.py:275-600, unchanged) through ``TieredEngine`` with the native
pool in accounting mode, the B200-measured prefill profile (profile.py) and
the measured host<->GPU bandwidth (bench ``kv_swap``), sweeping the GPU tier.
Reproduces the paper's hit-rate-driven TTFT reduction (PAPER.md:937-939,
1114-1118) on B200 numbers; p50 = ragsim's nearest-rank median
(simulator.py:177, 221-225).
"""

from __future__ import annotations

import dataclasses
import os
import tempfile

from . import cache
from ._ragsim import import_ragsim
from .pool import accounting_pool
from .workloads import Workload, make_stream, pool_blocks

import_ragsim()
from ragsim.config import RunConfig  # noqa: E402
from ragsim.cost_model import GIB_PER_S, save_profile_csv  # noqa: E402
from ragsim.simulator import measure_throughput, run as ragsim_run  # noqa: E402


def ttft_curve(w: Workload, profile, *, gpu_tiers, host_tier: int, n_requests: int = 3000,
               rate: float = 2.0, pcie_gbs: float = 55.0, stage_provider_fn=None,
               stage_interval_ms: float | None = None, decode_ms_per_token: float | None = None,
               seed: int = 0) -> list[dict]:
    trace, sizes = make_stream(w, n_requests, rate=rate, seed=seed)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "b200_profile.csv")
        save_profile_csv(profile, path)
        rows = []
        for cap in gpu_tiers:
            cfg = RunConfig(gpu_capacity_tokens=cap, host_capacity_tokens=host_tier,
                            k=w.k, profile_path=path,
                            kv_bytes_per_token=float(w.model.kv_bytes_per_token),
                            pcie_bandwidth_bytes_per_ms=pcie_gbs * 1e9 / 1e3, seed=seed,
                            **({"stage_interval_ms": stage_interval_ms}
                               if stage_interval_ms is not None else {}),
                            **({"decode_ms_per_token": decode_ms_per_token}
                               if decode_ms_per_token is not None else {}))
            pool = accounting_pool(pool_blocks(cap, w.block_tokens, sizes.values(), 8 * (w.k + 1)),
                                   pool_blocks(host_tier, w.block_tokens, sizes.values(), 0) or 1,
                                   w.block_tokens)
            sp = stage_provider_fn(trace, cfg) if stage_provider_fn else None
            report, _ = cache.run_tiered(cfg, trace, sizes, pool=pool, stage_provider=sp)
            a = report.aggregates()
            rows.append({"gpu_tier_tokens": cap, "host_tier_tokens": host_tier,
                         "doc_hit_rate": round(a["doc_hit_rate"], 4),
                         "p50_ttft_ms": round(a["median_ttft_ms"], 3),
                         "mean_ttft_ms": round(a["mean_ttft_ms"], 3),
                         "p99_ttft_ms": round(a["p99_ttft_ms"], 3),
                         "swap_outs": a["swap_outs"], "requests": a["requests"]})
    return rows


def slo_throughput(w: Workload, profile, *, gpu_tiers, host_tier: int, n_requests: int = 600,
                   pcie_gbs: float = 55.0, decode_ms_per_token: float | None = None,
                   slo_multiplier: float = 5.0, min_rate: float = 0.5, max_rate: float = 400.0,
                   iterations: int = 10, seed: int = 0) -> list[dict]:
    """RAG req/s in the paper's sense: the highest Poisson arrival rate
    whose mean TTFT stays within 5x the light-load mean TTFT, found by the reference's own
    bisection (measure_throughput, simulator.py:648-681) on B200-measured costs, per GPU
    tier (-> document hit rate)."""
    trace, sizes = make_stream(w, n_requests, rate=2.0, seed=seed)
    rows = []
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "b200_profile.csv")
        save_profile_csv(profile, path)
        for cap in gpu_tiers:
            cfg = RunConfig(gpu_capacity_tokens=cap, host_capacity_tokens=host_tier, k=w.k,
                            profile_path=path,
                            kv_bytes_per_token=float(w.model.kv_bytes_per_token),
                            pcie_bandwidth_bytes_per_ms=pcie_gbs * 1e9 / 1e3, seed=seed,
                            **({"decode_ms_per_token": decode_ms_per_token}
                               if decode_ms_per_token is not None else {}))
            rps = measure_throughput(cfg, trace, sizes, slo_multiplier, min_rate, max_rate,
                                     iterations=iterations)
            hit = ragsim_run(cfg, trace, sizes).aggregates()["doc_hit_rate"]
            rows.append({"gpu_tier_tokens": cap, "doc_hit_rate": round(hit, 4),
                         "req_per_s_at_slo": round(rps, 3)})
    return rows
