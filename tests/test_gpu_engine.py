"""The reference engine driven by the GPU retrieval kernel (a16/a18 rows).

ragsim's DSP controller (speculation.py:98-146) consumes the stages of
``GpuStageProvider`` (tcgen05 staged top-k).  The same engine run with stages
computed by the CPU oracle must give a byte-identical report: identical
candidate lists at every stage -> identical speculate/terminate/confirm
actions -> identical TTFTs.  The final stage must equal the trace's ground
truth (checked by ragsim itself, simulator.py:368-369).
"""

import dataclasses

import numpy as np
import pytest
import torch

from paper_2404_12457_b200._ragsim import ragsim_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")]


def test_engine_with_gpu_stages_matches_oracle_stages():
    from ragsim.config import RunConfig
    from ragsim.speculation import StagedRetrieval

    from oracle import topk_oracle
    from paper_2404_12457_b200 import cache, synth
    from paper_2404_12457_b200.pool import accounting_pool
    from paper_2404_12457_b200.retrieval import GpuStageProvider, synthetic_query_fn
    from tests.golden.make_golden import DESK, desk_trace

    trace, sizes = desk_trace(seed=0, duration_s=250.0, rate=0.25, pool=300)
    n_docs = 1500
    cfg = RunConfig(host_capacity_tokens=32768, stage_count=4, stage_interval_ms=50.0,
                    convergence_stage=2, prefill_chunk_ms=25.0, dsp=True, seed=0, validate=True,
                    **DESK)
    corpus = synth.corpus_int(n_docs, seed=0)
    qfn = synthetic_query_fn(seed=0, kind="int")  # exact scores: byte-identical reports
    gpu = GpuStageProvider(torch.from_numpy(corpus.astype(np.float32)).cuda().to(torch.bfloat16),
                           qfn, k=cfg.k, n_stages=cfg.stage_count,
                           stage_interval_ms=cfg.stage_interval_ms, trace=trace)

    def oracle_provider(req):
        q = qfn(req)[None]
        ids, _ = topk_oracle.staged_topk(corpus, q, cfg.k, cfg.stage_count)
        return StagedRetrieval(tuple(tuple(int(x) for x in st) for st in ids[0]),
                               cfg.stage_interval_ms)

    r_gpu, _ = cache.run_tiered(cfg, trace, sizes, pool=accounting_pool(4096, 8192, 16),
                                stage_provider=gpu)
    r_orc, _ = cache.run_tiered(cfg, trace, sizes, pool=accounting_pool(4096, 8192, 16),
                                stage_provider=oracle_provider)
    assert r_gpu.to_json(cfg) == r_orc.to_json(cfg)
    assert r_gpu.per_request_csv() == r_orc.per_request_csv()
    agg = r_gpu.aggregates()
    assert agg["speculations"] > 0  # DSP acted on the GPU's partial-scan candidates
    assert gpu.launches < 2 * len(trace)  # queries batched ahead (<= 64 per launch)
