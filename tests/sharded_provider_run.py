"""Run under torchrun (2 ranks, both on cuda:0, gloo): the package's sharded StageProvider
with the real kernels (rcb_retrieval_topk per shard, rcb_topk_merge_shards) drives a DSP
desk run on each rank's routed sub-trace.  Its report must be byte-identical to the same
run on an oracle provider computing the sharded staged top-k on the host
(oracle/topk_oracle.sharded_staged_topk), and every final stage must equal the unsharded
top-k.  Prints one JSON line per rank.  Invoked by tests/test_gpu_multirank.py."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from oracle import topk_oracle
    from paper_2404_12457_b200 import cache, synth  # puts ragsim (baseline/_ref) on the path
    from ragsim.config import RunConfig
    from ragsim.speculation import StagedRetrieval
    from paper_2404_12457_b200.dist import Dist, route, shard_bounds
    from paper_2404_12457_b200.pool import accounting_pool
    from paper_2404_12457_b200.retrieval import GpuStageProvider, synthetic_query_fn
    from tests.golden.make_golden import DESK, desk_trace

    torch.cuda.set_device(0)
    d = Dist().init("gloo")
    n_docs = 1500
    trace, sizes = desk_trace(seed=0, duration_s=250.0, rate=0.25, pool=300)
    sub = route(trace, d.rank, d.world)
    cfg = RunConfig(host_capacity_tokens=32768, stage_count=4, stage_interval_ms=50.0,
                    convergence_stage=2, prefill_chunk_ms=25.0, dsp=True, seed=0, validate=True,
                    **DESK)
    bounds = [shard_bounds(n_docs, r, d.world) for r in range(d.world)]
    lo, hi = bounds[d.rank]
    shards = [synth.corpus_int(b - a, seed=0, row_offset=a) for a, b in bounds]
    qfn = synthetic_query_fn(seed=0, kind="int")  # exact scores: byte-identical reports
    corpus = torch.from_numpy(shards[d.rank].astype(np.float32)).cuda().to(torch.bfloat16)
    sp = GpuStageProvider(corpus, qfn, k=cfg.k, n_stages=cfg.stage_count,
                          stage_interval_ms=cfg.stage_interval_ms, trace=sub, comm=d,
                          id_offset=lo, batch=16)
    full = np.concatenate(shards)
    finals_equal = True

    def oracle_provider(req):
        nonlocal finals_equal
        q = qfn(req)[None]
        ids, _ = topk_oracle.sharded_staged_topk(shards, [a for a, _ in bounds], q, cfg.k,
                                                 cfg.stage_count)
        one, _ = topk_oracle.staged_topk(full, q, cfg.k, cfg.stage_count)
        finals_equal &= bool(np.array_equal(ids[0, -1], one[0, -1]))
        return StagedRetrieval(tuple(tuple(int(x) for x in st) for st in ids[0]),
                               cfg.stage_interval_ms)

    r_gpu, _ = cache.run_tiered(cfg, sub, sizes, pool=accounting_pool(4096, 8192, 16),
                                stage_provider=sp)
    r_orc, _ = cache.run_tiered(cfg, sub, sizes, pool=accounting_pool(4096, 8192, 16),
                                stage_provider=oracle_provider)
    print(json.dumps({"rank": d.rank, "requests": len(sub),
                      "identical": r_gpu.to_json(cfg) == r_orc.to_json(cfg),
                      "finals_equal_unsharded": finals_equal,
                      "speculations": r_gpu.aggregates()["speculations"],
                      "launches": sp.launches}))
    d.barrier()
    d.close()


if __name__ == "__main__":
    main()
