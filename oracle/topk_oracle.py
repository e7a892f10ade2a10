"""ORACLE (test infrastructure only — never imported by the product path).

Exact staged inner-product top-k, restated on the CPU with numpy.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import it.

Reference anchoring:
* output contract = StagedRetrieval (ragsim speculation.py:33-59): one
  top-k tuple per stage, k constant across stages (:45-47), final stage =
  the ground truth the engine checks (simulator.py:368-369);
* stage s (0-based) of S = exact top-k over the first floor((s+1)*N/S) rows
  of the scan order — the "staged search" the paper's DSP consumes
  (PAPER.md:825-837); ragsim only synthesises it (speculation.py:149-194);
* ranking: score descending, then document id ascending.
The retrieval SCORES are unpinned by the reference (no embeddings in ragsim);
the IDS are pinned through the trace's ground-truth doc sequences
(workload.py:124-148) which the synthetic queries are built to reproduce.

With the integer-valued bf16 embeddings of paper_2404_12457_b200.synth every
inner product is an integer < 2^24, so float64 here and fp32 tensor-core
accumulation on the GPU are both exact: ids AND scores must match bit-exactly,
ties included.
"""

from __future__ import annotations

import numpy as np


def exact_scores(corpus: np.ndarray, queries: np.ndarray) -> np.ndarray:
    """[b, N] float64 scores (exact for the integer-valued synthetic corpus)."""
    return queries.astype(np.float64) @ corpus.astype(np.float64).T


def topk_rows(scores: np.ndarray, ids: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Top-k of one score vector by (score desc, id asc)."""
    n = scores.shape[0]
    if n == 0:
        return np.full(k, -1, dtype=np.int64), np.full(k, -np.inf)
    kk = min(k, n)
    thr = np.partition(scores, n - kk)[n - kk]
    cand = np.flatnonzero(scores >= thr)
    order = np.lexsort((ids[cand], -scores[cand]))[:kk]
    sel = cand[order]
    out_ids = np.full(k, -1, dtype=np.int64)
    out_sc = np.full(k, -np.inf)
    out_ids[:kk] = ids[sel]
    out_sc[:kk] = scores[sel]
    return out_ids, out_sc


def staged_topk(corpus: np.ndarray, queries: np.ndarray, k: int, n_stages: int,
                id_offset: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Returns ids int64 [b, S, k] and scores float64 [b, S, k]."""
    n = corpus.shape[0]
    scores = exact_scores(corpus, queries)
    ids = np.arange(n, dtype=np.int64) + id_offset
    b = queries.shape[0]
    out_ids = np.empty((b, n_stages, k), dtype=np.int64)
    out_sc = np.empty((b, n_stages, k))
    for qi in range(b):
        for s in range(n_stages):
            bound = (n * (s + 1)) // n_stages
            out_ids[qi, s], out_sc[qi, s] = topk_rows(scores[qi, :bound], ids[:bound], k)
    return out_ids, out_sc


def sharded_staged_topk(shards: list[np.ndarray], offsets: list[int], queries: np.ndarray,
                        k: int, n_stages: int) -> tuple[np.ndarray, np.ndarray]:
    """Corpus split across G shards: stage s = top-k over the union of every
    shard's first (s+1)/S rows (the sharded scan order)."""
    per = [staged_topk(c, queries, k, n_stages, off) for c, off in zip(shards, offsets)]
    b = queries.shape[0]
    out_ids = np.empty((b, n_stages, k), dtype=np.int64)
    out_sc = np.empty((b, n_stages, k))
    for qi in range(b):
        for s in range(n_stages):
            ids = np.concatenate([p[0][qi, s] for p in per])
            sc = np.concatenate([p[1][qi, s] for p in per])
            keep = ids >= 0
            out_ids[qi, s], out_sc[qi, s] = topk_rows(sc[keep], ids[keep], k)
    return out_ids, out_sc
