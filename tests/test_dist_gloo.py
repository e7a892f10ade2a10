"""Multi-GPU host logic on CPU: world_size-2 gloo.

* corpus shards + gather/merge: every rank scans its contiguous shard for ALL
  ranks' queries (oracle scan on CPU), the per-shard staged lists are
  all-gathered through ``Dist`` and merged (score desc, id asc); each rank's
  slice must equal the sharded-scan oracle, and the final stage must equal
  the unsharded exact top-k;
* data-parallel replicas: requests routed by ``id mod world`` partition the
  trace, and each rank's TieredEngine (reference decisions + native pool in
  accounting mode) reproduces ragsim.run on its routed sub-trace byte-for-byte.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2404_12457_b200._ragsim import ragsim_available

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _merge(ids, scores, k):
    """[G, nq, S, k] -> [nq, S, k] with the device merge's ordering rule."""
    from oracle.topk_oracle import topk_rows

    g, nq, S, _ = ids.shape
    out = np.empty((nq, S, k), dtype=np.int64)
    for q in range(nq):
        for s in range(S):
            i = ids[:, q, s].reshape(-1)
            sc = scores[:, q, s].reshape(-1)
            keep = i >= 0
            out[q, s] = topk_rows(sc[keep], i[keep], k)[0]
    return out


def _worker(rank, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(WORLD), LOCAL_RANK=str(rank))
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import topk_oracle
    from paper_2404_12457_b200 import synth
    from paper_2404_12457_b200.dist import Dist, route, shard_bounds

    d = Dist().init("gloo")
    try:
        n, k, S, per_rank = 3001, 3, 4, 5
        lo, hi = shard_bounds(n, rank, WORLD)
        shard = synth.corpus_int(hi - lo, seed=7, row_offset=lo)
        q_local = np.random.default_rng(rank).integers(-50, 51, size=(per_rank, synth.EMB_DIM))
        allq = d.all_gather(torch.from_numpy(q_local.astype(np.float64))).reshape(-1, synth.EMB_DIM)
        allq = allq.numpy()
        ids, sc = topk_oracle.staged_topk(shard, allq, k, S, id_offset=lo)
        gi = d.all_gather(torch.from_numpy(ids)).numpy()
        gs = d.all_gather(torch.from_numpy(sc)).numpy()
        merged = _merge(gi, gs, k)[rank * per_rank:(rank + 1) * per_rank]
        bounds = [shard_bounds(n, r, WORLD) for r in range(WORLD)]
        shards = [synth.corpus_int(b - a, seed=7, row_offset=a) for a, b in bounds]
        exp, _ = topk_oracle.sharded_staged_topk(shards, [a for a, _ in bounds], allq, k, S)
        assert np.array_equal(merged, exp[rank * per_rank:(rank + 1) * per_rank])
        full, _ = topk_oracle.staged_topk(np.concatenate(shards), allq, k, S)
        assert np.array_equal(exp[:, -1], full[:, -1])  # final stage = unsharded top-k

        from paper_2404_12457_b200._ragsim import ragsim_available

        if ragsim_available():
            from ragsim.config import RunConfig
            from ragsim.simulator import run

            from paper_2404_12457_b200 import cache
            from paper_2404_12457_b200.pool import accounting_pool
            from tests.golden.make_golden import DESK, desk_trace

            trace, sizes = desk_trace(seed=3, duration_s=150.0, rate=0.6, pool=300)
            sub = route(trace, rank, WORLD)
            counts = d.all_gather(torch.tensor([len(sub)])).reshape(-1)
            assert int(counts.sum()) == len(trace)
            cfg = RunConfig(host_capacity_tokens=24576, seed=3, **DESK)
            ref = run(cfg, sub, sizes)
            rep, _ = cache.run_tiered(cfg, sub, sizes, pool=accounting_pool(2048, 4096, 16))
            assert rep.to_json(cfg) == ref.to_json(cfg)
        d.barrier()
        results.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        results.put((rank, repr(exc)))
    finally:
        d.close()


def test_two_rank_gloo_shards_and_replicas():
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, results)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(results.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    assert got == {0: "ok", 1: "ok"}, got


def _oracle_scan(corpus_np):
    from oracle import topk_oracle

    def scan(corpus, q, k, S, off):
        ids, sc = topk_oracle.staged_topk(corpus_np, q.float().numpy().astype(np.float64), k, S,
                                          id_offset=off)
        return torch.from_numpy(ids), torch.from_numpy(sc.astype(np.float32))

    return scan


def _oracle_merge(gi, gs):
    k = gi.shape[-1]
    return torch.from_numpy(_merge(gi.numpy(), gs.numpy(), k)), None


def _provider_worker(rank, port, results):
    """The package's sharded StageProvider (ShardedRetriever: query all-gather, per-shard
    scan, list all-gather, merge) driving a DSP desk run on each rank's routed sub-trace.
    The scan and merge are the oracle's here (no GPU); the collectives, padding,
    lockstep rounds and routing are the product's."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(WORLD), LOCAL_RANK=str(rank))
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from ragsim.config import RunConfig
    from ragsim.speculation import StagedRetrieval

    from oracle import topk_oracle
    from paper_2404_12457_b200 import cache, synth
    from paper_2404_12457_b200.dist import Dist, route, shard_bounds
    from paper_2404_12457_b200.pool import accounting_pool
    from paper_2404_12457_b200.retrieval import GpuStageProvider, ShardedRetriever, synthetic_query_fn
    from tests.golden.make_golden import DESK, desk_trace

    d = Dist().init("gloo")
    try:
        n_docs = 1500
        trace, sizes = desk_trace(seed=0, duration_s=200.0, rate=0.3, pool=300)
        sub = route(trace, rank, WORLD)
        cfg = RunConfig(host_capacity_tokens=32768, stage_count=4, stage_interval_ms=50.0,
                        convergence_stage=2, prefill_chunk_ms=25.0, dsp=True, seed=0,
                        validate=True, **DESK)
        lo, hi = shard_bounds(n_docs, rank, WORLD)
        shard = synth.corpus_int(hi - lo, seed=0, row_offset=lo)
        qfn = synthetic_query_fn(seed=0, kind="int")
        retr = ShardedRetriever(torch.from_numpy(shard.astype(np.float32)), lo, cfg.k,
                                cfg.stage_count, d, batch=8, scan=_oracle_scan(shard),
                                merge=_oracle_merge)
        sp = GpuStageProvider(retr.corpus, qfn, k=cfg.k, n_stages=cfg.stage_count,
                              stage_interval_ms=cfg.stage_interval_ms, trace=sub, retriever=retr)
        bounds = [shard_bounds(n_docs, r, WORLD) for r in range(WORLD)]
        shards = [synth.corpus_int(b - a, seed=0, row_offset=a) for a, b in bounds]
        full = np.concatenate(shards)

        def oracle_provider(req):
            q = qfn(req)[None]
            ids, _ = topk_oracle.sharded_staged_topk(shards, [a for a, _ in bounds], q, cfg.k,
                                                     cfg.stage_count)
            one, _ = topk_oracle.staged_topk(full, q, cfg.k, cfg.stage_count)
            assert np.array_equal(ids[0, -1], one[0, -1])  # final stage = 1 shard
            return StagedRetrieval(tuple(tuple(int(x) for x in st) for st in ids[0]),
                                   cfg.stage_interval_ms)

        r_sh, _ = cache.run_tiered(cfg, sub, sizes, pool=accounting_pool(4096, 8192, 16),
                                   stage_provider=sp)
        r_or, _ = cache.run_tiered(cfg, sub, sizes, pool=accounting_pool(4096, 8192, 16),
                                   stage_provider=oracle_provider)
        assert r_sh.to_json(cfg) == r_or.to_json(cfg)
        assert r_sh.aggregates()["speculations"] > 0
        d.barrier()
        results.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        import traceback

        results.put((rank, traceback.format_exc()[-1500:]))
    finally:
        d.close()


@pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")
def test_two_rank_sharded_stage_provider_dsp_run():
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_provider_worker, args=(r, port, results)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(results.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    assert got == {0: "ok", 1: "ok"}, got


def test_shard_bounds_and_route_partition():
    from paper_2404_12457_b200.dist import route, shard_bounds

    for n in (1, 7, 100_000, 10_000_000):
        for world in (1, 2, 4, 8):
            b = [shard_bounds(n, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))

    class R:
        def __init__(self, i):
            self.id = i

    reqs = [R(i) for i in range(37)]
    parts = [route(reqs, r, 4) for r in range(4)]
    assert sorted(x.id for p in parts for x in p) == list(range(37))


def test_slo_throughput_rises_with_hit_rate():
    """ragsim's measure_throughput on a profile: more GPU tier -> more doc hits -> a
    higher arrival rate fits the 5x TTFT SLO (the paper's throughput metric)."""
    from paper_2404_12457_b200._ragsim import ragsim_available

    if not ragsim_available():
        pytest.skip("ragsim not importable")
    from ragsim.cost_model import synthetic_profile

    from paper_2404_12457_b200.ttft import slo_throughput
    from paper_2404_12457_b200.workloads import WORKLOADS

    qw = WORKLOADS["mistral7b-100k-qpool"]
    lo, hi = slo_throughput(qw, synthetic_profile(), gpu_tiers=[2200, qw.gpu_capacity_tokens],
                            host_tier=qw.host_capacity_tokens, n_requests=300,
                            decode_ms_per_token=5.0, iterations=8)
    assert hi["doc_hit_rate"] > lo["doc_hit_rate"] + 0.3
    assert hi["req_per_s_at_slo"] > lo["req_per_s_at_slo"]
