"""Hardware-in-the-loop curves for the bench: TTFT vs hit rate and req/s at the 5x TTFT SLO
with every admitted prefill EXECUTED on the GPU (TimedEngine).

* ``timed_ttft_curve``: the reference's engine (decisions, queue, DSP, virtual clock,
  simulator.py:275-600) on a trace, per GPU tier; each admission's prefill runs the
  random-init model (cuBLAS GEMMs + our RoPE/KV-write and prefix-prefill kernels) on its
  real block table in a device pool of the tier's size, and its CUDA-event time advances
  the clock.  The profile-driven run of the same trace is reported beside it.
* ``timed_slo_throughput``: ragsim's ``measure_throughput`` bisection (simulator.py:
  648-681: the highest Poisson rate whose mean TTFT stays within 5x the light-load mean)
  where every probe is a timed run.

One model instance serves every run (weights built once); each run gets a fresh pool over
one preallocated HBM buffer (``gpu_base``), so runs are independent.
"""

from __future__ import annotations

import time

import torch

from . import cache
from .pool import BlockPool, accounting_pool
from .timed import ModelExecutor, run_timed
from .workloads import make_stream, pool_blocks

from ragsim.simulator import scale_trace  # noqa: E402  (ragsim is on the path via .cache)


class TimedRunner:
    """Model weights + one HBM pool buffer for timed runs at GPU tiers <= max_tier."""

    def __init__(self, w, max_tier: int, host_tier: int, *, swap_in: str = "modeled",
                 swap_mode: int | None = None, seed: int = 0) -> None:
        from . import _lib
        from .model import DIMS, init_weights

        self.w = w
        s = w.model
        self.dims = DIMS[w.shape]
        self.weights = init_weights(self.dims, seed=seed)
        self.swap_in = swap_in
        self.swap_mode = _lib.RCB_SWAP_DMA if swap_mode is None else swap_mode
        self.host_tier = host_tier
        self.block_bytes = w.block_tokens * s.kv_bytes_per_token
        self.max_tier = max_tier
        self._buf = None
        self._buf_blocks = 0

    def _pool(self, cap: int, sizes):
        w, s = self.w, self.w.model
        ng = pool_blocks(cap, w.block_tokens, sizes.values(), 8 * (w.k + 1))
        nh = pool_blocks(self.host_tier, w.block_tokens, sizes.values(), 0) or 1
        if ng > self._buf_blocks:
            self._buf = None
            torch.cuda.empty_cache()
            self._buf = torch.empty(ng * self.block_bytes, dtype=torch.uint8, device="cuda")
            self._buf_blocks = ng
        return BlockPool(ng, nh, block_tokens=w.block_tokens, n_layers=s.n_layers,
                         n_kv_heads=s.n_kv_heads, head_dim=s.head_dim, swap_mode=self.swap_mode,
                         gpu_base=self._buf.data_ptr()), (ng, nh)

    def run(self, cfg, trace, sizes):
        pool, _ = self._pool(cfg.gpu_capacity_tokens, sizes)
        ex = ModelExecutor(pool, self.w.shape, swap_in=self.swap_in, weights=self.weights,
                           layers_per_group=1)
        try:
            rep, engine = run_timed(cfg, trace, sizes, pool=pool, executor=ex)
            pool.sync()
            torch.cuda.synchronize()
            stats = pool.stats()
        finally:
            pool.close()
        return rep, engine, stats

    def close(self) -> None:
        self._buf = None
        self.weights = None
        torch.cuda.empty_cache()


def _cfg(w, cap, host, prof_path, dec_ms, stage_ms, pcie_gbs, **kw):
    from ragsim.config import RunConfig

    return RunConfig(gpu_capacity_tokens=cap, host_capacity_tokens=host, k=w.k,
                     profile_path=prof_path, decode_ms_per_token=dec_ms,
                     stage_interval_ms=stage_ms, pcie_bandwidth_bytes_per_ms=pcie_gbs * 1e6,
                     kv_bytes_per_token=float(w.model.kv_bytes_per_token), seed=w.seed, **kw)


def timed_ttft_curve(runner: TimedRunner, tiers, *, prof_path: str, dec_ms: float,
                     stage_ms: float, pcie_gbs: float, n_requests: int = 400,
                     rate: float = 2.0) -> list[dict]:
    w = runner.w
    trace, sizes = make_stream(w, n_requests, rate=rate)
    rows = []
    for cap in tiers:
        cfg = _cfg(w, cap, runner.host_tier, prof_path, dec_ms, stage_ms, pcie_gbs)
        t0 = time.perf_counter()
        rep, engine, st = runner.run(cfg, trace, sizes)
        ng = pool_blocks(cap, w.block_tokens, sizes.values(), 8 * (w.k + 1))
        nh = pool_blocks(runner.host_tier, w.block_tokens, sizes.values(), 0) or 1
        prof_rep, _ = cache.run_tiered(cfg, trace, sizes,
                                       pool=accounting_pool(ng, nh, w.block_tokens))
        a, b = rep.aggregates(), prof_rep.aggregates()
        ratio = sorted(m / p for _, _, _, p, m in engine.measured if p > 0)
        rows.append({"gpu_tier_tokens": cap, "doc_hit_rate": round(a["doc_hit_rate"], 4),
                     "p50_ttft_ms": round(a["median_ttft_ms"], 3),
                     "mean_ttft_ms": round(a["mean_ttft_ms"], 3),
                     "p99_ttft_ms": round(a["p99_ttft_ms"], 3),
                     "profile_p50_ttft_ms": round(b["median_ttft_ms"], 3),
                     "prefills_executed": len(engine.measured),
                     "measured_over_profile_median": round(ratio[len(ratio) // 2], 3) if ratio else None,
                     "swap_out_bytes": st["d2h_bytes"], "swap_in_bytes": st["h2d_bytes"],
                     "seconds": round(time.perf_counter() - t0, 1)})
    return rows


def timed_slo_throughput(runner: TimedRunner, cap: int, *, prof_path: str, dec_ms: float,
                         stage_ms: float, pcie_gbs: float, n_requests: int = 300,
                         slo_multiplier: float = 5.0, min_rate: float = 0.5,
                         max_rate: float = 400.0, iterations: int = 7) -> dict:
    """simulator.py:648-681 with timed probes (each probe = one TimedEngine run)."""
    w = runner.w
    trace, sizes = make_stream(w, n_requests, rate=2.0)
    cfg = _cfg(w, cap, runner.host_tier, prof_path, dec_ms, stage_ms, pcie_gbs)
    span_ms = max(r.arrival_ms for r in trace) or 1.0
    base_rate = len(trace) / (span_ms / 1000.0)
    probes = []

    def mean_ttft(rate: float):
        rep, _, _ = runner.run(cfg, scale_trace(trace, base_rate / rate), sizes)
        a = rep.aggregates()
        probes.append((round(rate, 3), round(a["mean_ttft_ms"], 3)))
        return a["mean_ttft_ms"], a["doc_hit_rate"]

    t0 = time.perf_counter()
    light, hit = mean_ttft(min_rate)
    slo = slo_multiplier * light
    if mean_ttft(max_rate)[0] <= slo:
        best = max_rate
    else:
        lo, hi = min_rate, max_rate
        for _ in range(iterations):
            mid = (lo + hi) / 2.0
            if mean_ttft(mid)[0] <= slo:
                lo = mid
            else:
                hi = mid
        best = lo
    return {"gpu_tier_tokens": cap, "doc_hit_rate_light_load": round(hit, 4),
            "req_per_s_at_slo": round(best, 3), "slo_ms": round(slo, 3),
            "probes": probes, "iterations": iterations, "requests": n_requests,
            "seconds": round(time.perf_counter() - t0, 1)}
