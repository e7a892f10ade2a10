"""The N > 1 path of bench.py on one GPU: two ranks (gloo plumbing, both on cuda:0).

Exercises what the 8-GPU run shards: requests routed id mod G to
per-rank knowledge-tree replicas, the corpus split into row shards, queries
all-gathered, every rank scanning its shard, per-shard staged top-k lists
all-gathered and merged on device (rcb_topk_merge_shards), max-over-ranks timing.
The merged final stage must reproduce every request's ground-truth documents.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_bench_on_one_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "2",
           "--single-device", "--backend", "gloo", "--steps", "2", "--warmup", "3", "--no-ttft",
           "--no-cpu-baseline", "--gpu-tier-tokens", "50000", "--cache-warm-steps", "5"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]  # rank 0 prints the one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["retrieval_final_stage_matches_ground_truth"]
    assert d["e2e"]["retrieval_matches_ground_truth"]


def test_two_rank_sharded_stage_provider_on_one_gpu():
    """GpuStageProvider(comm=...) with the real kernels: per-rank corpus shards, lockstep
    query all-gather, shard scans, list all-gather and device merge under a DSP run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29543",
           os.path.join("tests", "sharded_provider_run.py")]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, [l for l in res.stderr.splitlines() if "Error" in l][:10]
    rows = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert sorted(r["rank"] for r in rows) == [0, 1]
    for r in rows:
        assert r["identical"] and r["finals_equal_unsharded"], r
        assert r["speculations"] > 0 and r["requests"] > 0


def test_two_rank_peer_exchange_matches_allgather():
    """The per-shard lists meet over peer memory (CUDA IPC windows, push + epoch flags +
    device merge): bit-identical to the all-gather exchange over several calls."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29545",
           os.path.join("tests", "peer_exchange_run.py")]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    rows = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert sorted(r["rank"] for r in rows) == [0, 1]
    for r in rows:
        assert r["exchange"] == "p2p" and r["identical"] and r["epoch"] == r["calls"], r
