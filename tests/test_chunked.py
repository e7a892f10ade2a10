"""Chunked prefill with real termination (simulator.py:408-425, 507-510).

The suffix runs in the reference's chunk count, one chunk per iteration boundary, with
alpha growing per chunk (each chunk attends the cached prefix plus the earlier chunks'
pages).  A speculation terminated mid-prefill stops launching chunks.

CPU: a fake chunked executor charging the reference's own chunk length makes TimedEngine
reproduce ragsim.run's TTFTs and aggregates (the chunk bookkeeping is the reference's).
GPU: chunked logits == unchunked logits (and the fp32 oracle) within 1e-2; a DSP run
where terminated speculations skip their remaining chunks.
"""

import types

import numpy as np
import pytest

from paper_2404_12457_b200._ragsim import ragsim_available

pytestmark = pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")


def _dsp_desk(chunk_ms, stage_ms=50.0):
    from ragsim.config import RunConfig

    from tests.golden.make_golden import DESK, desk_trace, pool_geometry

    trace, sizes = desk_trace(seed=0, duration_s=300.0, rate=0.25, pool=300)
    cfg = RunConfig(host_capacity_tokens=32768, stage_count=4, stage_interval_ms=stage_ms,
                    convergence_stage=2, prefill_chunk_ms=chunk_ms, dsp=True, seed=0,
                    validate=True, **DESK)
    return cfg, trace, sizes, pool_geometry(cfg, sizes)


class _ChunkedProfileExecutor:
    """Charges ragsim's own chunk length (simulator.py:507-509) per executed chunk."""

    chunked = True

    def __init__(self):
        self.last_ms = 0.0
        self.last_transfer_ms = 0.0
        self.chunks_run = 0

    def on_admit(self, engine, gen, blocks, valid):
        gen.exec_state = {"n": gen.chunks_left}
        self.chunk = gen.chunk_ms
        gen.exec_state["chunk"] = gen.chunk_ms
        self.last_ms = gen.chunk_ms
        self.chunks_run += 1

    def run_chunk(self, gen, c):
        assert 0 < c < gen.exec_state["n"]
        self.chunks_run += 1
        return gen.exec_state["chunk"]


def test_chunk_bookkeeping_reproduces_reference_timing():
    from ragsim.simulator import run

    from paper_2404_12457_b200.pool import accounting_pool
    from paper_2404_12457_b200.timed import run_timed

    cfg, trace, sizes, (ng, nh) = _dsp_desk(chunk_ms=5.0)
    ref = run(cfg, trace, sizes)
    ex = _ChunkedProfileExecutor()
    rep, engine = run_timed(cfg, trace, sizes, pool=accounting_pool(ng, nh, 16), executor=ex)
    a, b = ref.aggregates(), rep.aggregates()
    for key in ("requests", "doc_hit_rate", "speculations", "gpu_evictions", "swap_outs"):
        assert a[key] == b[key], key
    for key in ("mean_ttft_ms", "median_ttft_ms", "p99_ttft_ms", "mean_non_overlap_ms"):
        assert abs(a[key] - b[key]) < 1e-6 * max(1.0, abs(a[key])), key
    assert engine.planned_chunks > len(trace)  # several chunks per prefill
    assert engine.skipped_chunks > 0  # terminated speculations stopped early
    assert ex.chunks_run + engine.skipped_chunks == engine.planned_chunks


@pytest.mark.gpu
def test_chunked_prefill_logits_match_unchunked_and_oracle():
    import torch

    from oracle import model_oracle
    from paper_2404_12457_b200.model import DIMS
    from paper_2404_12457_b200.pool import BlockPool
    from paper_2404_12457_b200.timed import ModelExecutor, doc_tokens

    dims = DIMS["tiny"]
    sizes = {1: 300, 2: 170, 3: 513}
    outs = {}
    for n_chunks in (1, 4):
        pool = BlockPool(256, 0, block_tokens=16, n_layers=2, n_kv_heads=4, head_dim=64)
        ex = ModelExecutor(pool, "tiny", chunked=True)
        engine = types.SimpleNamespace(sizes=sizes)
        # doc 1 cached (written by an earlier unchunked prefill), docs 2, 3 + prompt missing
        first = types.SimpleNamespace(
            pool_ctx=types.SimpleNamespace(seg_docs=[1, None]), request=types.SimpleNamespace(
                id=7, prompt_tokens=32), matched_nodes=[], alpha=0, beta=332, chunks_left=1)
        pool.gen_reserve(0, [300, 32])
        blocks, valid = pool.block_table([], 0)
        ex.on_admit(engine, first, blocks, valid)
        pool.node_adopt(1, 0, 0)  # the committed node takes the pages its prefill wrote
        pool.gen_release(0)
        node = types.SimpleNamespace(size=300)
        gen = types.SimpleNamespace(
            pool_ctx=types.SimpleNamespace(seg_docs=[2, 3, None]), request=types.SimpleNamespace(
                id=9, prompt_tokens=32), matched_nodes=[node], alpha=300, beta=170 + 513 + 32,
            chunks_left=n_chunks)
        pool.gen_reserve(1, [170, 513, 32])
        blocks, valid = pool.block_table([1], 1)
        ex.on_admit(engine, gen, blocks, valid)
        for c in range(1, n_chunks):
            ex.run_chunk(gen, c)
        assert ex.chunks_run == 1 + n_chunks
        outs[n_chunks] = ex.last_logits[0].float().cpu()
        seq = torch.from_numpy(np.concatenate([doc_tokens(d, sizes[d], dims.vocab, 0)
                                               for d in (1, 2, 3)]
                                              + [doc_tokens(-10, 32, dims.vocab, 0)]))
        ref = model_oracle.forward_full(ex.w, dims, seq)[-1]
        assert (outs[n_chunks] - ref).abs().max().item() <= 1e-2
        pool.close()
    assert (outs[1] - outs[4]).abs().max().item() <= 1e-2


@pytest.mark.gpu
def test_terminated_speculations_launch_fewer_chunks():
    import torch

    from paper_2404_12457_b200.pool import BlockPool
    from paper_2404_12457_b200.timed import ModelExecutor, run_timed

    # B200 runs the tiny model's chunks in ~0.1-0.3 ms: retrieval stages 0.25 ms apart so that
    # stale speculations are terminated while their prefill is still running
    cfg, trace, sizes, (ng, nh) = _dsp_desk(chunk_ms=5.0, stage_ms=0.25)
    pool = BlockPool(ng, nh, block_tokens=16, n_layers=2, n_kv_heads=4, head_dim=64)
    ex = ModelExecutor(pool, "tiny", chunked=True)
    rep, engine = run_timed(cfg, trace, sizes, pool=pool, executor=ex)
    pool.sync()
    torch.cuda.synchronize()
    assert rep.aggregates()["requests"] == len(trace)
    assert engine.planned_chunks > len(engine.measured)  # prefills ran in several chunks
    assert engine.skipped_chunks > 0
    # the admissions' chunk 0 plus every later chunk that was not skipped
    assert ex.chunks_run + engine.skipped_chunks == engine.planned_chunks
    pool.close()
