"""Run under torchrun (2 ranks, both on cuda:0, gloo plumbing): the peer-memory list
exchange (kernels.PeerExchange: CUDA IPC windows, push + epoch flags + merge) against the
all-gather exchange on the same shards and queries, several calls (both window parities).
Prints one JSON line per rank.  Invoked by tests/test_gpu_multirank.py."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    from paper_2404_12457_b200 import synth
    from paper_2404_12457_b200.dist import Dist, shard_bounds
    from paper_2404_12457_b200.retrieval import ShardedRetriever

    torch.cuda.set_device(0)
    d = Dist().init("gloo")
    n_rows, batch, k, S = 20_000, 48, 4, 4
    lo, hi = shard_bounds(n_rows, d.rank, d.world)
    shard = synth.corpus_device(hi - lo, seed=3, row_offset=lo)
    p2p = ShardedRetriever(shard, lo, k, S, d, batch=batch, exchange="p2p")
    ag = ShardedRetriever(shard, lo, k, S, d, batch=batch, exchange="allgather")
    g = torch.Generator(device="cuda").manual_seed(11 + d.rank)
    same = True
    calls = 5
    for _ in range(calls):
        q = torch.randn((batch, shard.shape[1]), generator=g, device="cuda").to(torch.bfloat16)
        i1, s1 = p2p(q, with_scores=True)
        i2, s2 = ag(q, with_scores=True)
        same &= bool(torch.equal(i1, i2)) and bool(torch.equal(s1, s2))
    torch.cuda.synchronize()
    p2p.px.check_timeout()
    p2p.pq.check_timeout()
    print(json.dumps({"rank": d.rank, "exchange": p2p.exchange, "calls": calls,
                      "identical": same, "epoch": p2p.px.epoch}))
    d.barrier()
    p2p.px.close()
    p2p.pq.close()
    d.close()


if __name__ == "__main__":
    main()
