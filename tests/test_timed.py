"""Hardware-in-the-loop engine.

CPU: with an executor that returns the profile's own interpolation, TimedEngine's
interception of the first-chunk scheduling must reproduce ragsim.run byte for byte
(simulator.py:481-514).  GPU: the tiny model's real prefill (GEMMs + our kernels on each
generation's block table in the device pool, swaps included) drives the virtual clock.
"""

import pytest

from paper_2404_12457_b200._ragsim import ragsim_available

pytestmark = pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")


def _desk():
    from ragsim.config import RunConfig

    from tests.golden.make_golden import DESK, desk_trace, pool_geometry

    trace, sizes = desk_trace(seed=3, duration_s=200.0, rate=0.6, pool=400)
    cfg = RunConfig(host_capacity_tokens=24576, dsp=True, stage_count=4, validate=True,
                    prefill_chunk_ms=25.0, **DESK)
    return cfg, trace, sizes, pool_geometry(cfg, sizes)


def test_timed_engine_with_profile_executor_reproduces_reference():
    from ragsim.simulator import run

    from paper_2404_12457_b200.pool import accounting_pool
    from paper_2404_12457_b200.timed import ProfileExecutor, run_timed

    cfg, trace, sizes, (ng, nh) = _desk()
    ref = run(cfg, trace, sizes)
    rep, engine = run_timed(cfg, trace, sizes, pool=accounting_pool(ng, nh, 16),
                            executor=ProfileExecutor())
    assert rep.to_json(cfg) == ref.to_json(cfg)
    assert rep.per_request_csv() == ref.per_request_csv()
    assert len(engine.measured) >= len(trace)
    assert all(m == p for _, _, _, p, m in engine.measured)


@pytest.mark.gpu
def test_timed_engine_runs_real_prefills():
    import torch

    from paper_2404_12457_b200.pool import BlockPool
    from paper_2404_12457_b200.timed import ModelExecutor, run_timed

    cfg, trace, sizes, (ng, nh) = _desk()
    pool = BlockPool(ng, nh, block_tokens=16, n_layers=2, n_kv_heads=4, head_dim=64)
    ex = ModelExecutor(pool, "tiny")
    rep, engine = run_timed(cfg, trace, sizes, pool=pool, executor=ex)
    pool.sync()
    torch.cuda.synchronize()
    agg = rep.aggregates()
    assert agg["requests"] == len(trace)
    assert len(engine.measured) >= len(trace)
    assert all(m > 0 for *_, m in engine.measured)
    st = pool.stats()
    assert st["swap_out_blocks"] > 0  # the host tier was exercised with real copies
    # a cached-prefix prefill of the same beta is no slower than computing the prefix too
    hits = [m for _, a, b, _, m in engine.measured if a > 0 and b <= 64]
    misses = [m for _, a, b, _, m in engine.measured if a == 0 and b > 512]
    if hits and misses:
        assert sorted(hits)[len(hits) // 2] < sorted(misses)[len(misses) // 2]
    pool.close()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["serial", "layered"])
def test_timed_engine_executes_swap_ins(mode):
    """The measured swap-in modes: the host-tier hits' H2D runs inside the timed region
    (serially, or per layer group overlapping the prefill) and is charged as prefill time."""
    import torch

    from paper_2404_12457_b200 import _lib
    from paper_2404_12457_b200.pool import BlockPool
    from paper_2404_12457_b200.timed import ModelExecutor, run_timed

    cfg, trace, sizes, (ng, nh) = _desk()
    pool = BlockPool(ng, nh, block_tokens=16, n_layers=2, n_kv_heads=4, head_dim=64,
                     swap_mode=_lib.RCB_SWAP_DMA)
    ex = ModelExecutor(pool, "tiny", swap_in=mode, layers_per_group=1)
    rep, engine = run_timed(cfg, trace, sizes, pool=pool, executor=ex)
    pool.sync()
    torch.cuda.synchronize()
    assert rep.aggregates()["requests"] == len(trace)
    assert pool.stats()["swap_in_blocks"] > 0
    # every admission's transfer was executed, not modelled
    assert all(t == 0.0 for _, _, t, _ in engine.critical)
    assert any(mt > 0 for _, mt, _, _ in engine.critical)  # some admissions had host hits
    pool.close()


@pytest.mark.gpu
def test_timed_curves_and_slo_throughput_tiny():
    """bench.py's hardware-in-the-loop block on the tiny workload: more GPU tier -> more doc
    hits -> lower executed TTFT; the timed SLO bisection returns a rate within bounds."""
    import os

    from ragsim.cost_model import save_profile_csv, synthetic_profile

    from paper_2404_12457_b200.timed_curves import (TimedRunner, timed_slo_throughput,
                                                    timed_ttft_curve)
    from paper_2404_12457_b200.workloads import WORKLOADS

    w = WORKLOADS["tiny-1k"]
    path = os.path.join("/tmp", "tiny_profile_test.csv")
    save_profile_csv(synthetic_profile(), path)
    runner = TimedRunner(w, 20_000, 0)
    kw = dict(prof_path=path, dec_ms=2.0, stage_ms=1.0, pcie_gbs=50.0)
    rows = timed_ttft_curve(runner, [5000, 20_000], n_requests=150, **kw)
    assert rows[1]["doc_hit_rate"] > rows[0]["doc_hit_rate"]
    assert all(r["prefills_executed"] >= 150 for r in rows)
    slo = timed_slo_throughput(runner, 20_000, n_requests=80, iterations=2, max_rate=100.0, **kw)
    assert 0.5 <= slo["req_per_s_at_slo"] <= 100.0 and len(slo["probes"]) >= 2
    runner.close()
