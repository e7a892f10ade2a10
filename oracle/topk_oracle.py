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

Two parity regimes:
* INTEGER corpus (synth.corpus_int): every inner product is an integer < 2^24,
  so float64 here and fp32 tensor-core accumulation on the GPU are both exact:
  ids AND scores must match bit-exactly, ties included (`staged_topk`).
* REAL corpus (synth.corpus_f32, unit-norm bf16 rows): fp32 accumulation
  differs from float64 by at most ``acc_bound`` per score.  A stage whose
  float64 top-(k+1) has every adjacent gap above 2*bound has a unique answer,
  and the GPU ids must equal it bit-exactly; the other stages ("ambiguous",
  counted and reported) must still be a top-k within the bound
  (`check_topk_tolerant`).  Separately, the kernel's selection is bit-exact
  against its own fp32 scores (rcb_retrieval_scores) through `staged_topk`.
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
    return staged_topk_from_scores(exact_scores(corpus, queries), k, n_stages, id_offset)


def staged_topk_from_scores(scores: np.ndarray, k: int, n_stages: int,
                            id_offset: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Staged top-k of a given [b, N] score matrix (e.g. the kernel's own fp32 scores,
    which pins its selection logic bit for bit)."""
    b, n = scores.shape
    scores = scores.astype(np.float64)
    ids = np.arange(n, dtype=np.int64) + id_offset
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


def acc_bound(queries: np.ndarray, corpus_max_norm: float = 1.0 + 2.0 ** -8) -> np.ndarray:
    """[b] bound on |fp32-accumulated score - exact score| for a dim-term bf16 dot product.

    Products of two bf16 values are exact in fp32; summing dim of them in fp32 (any
    order, round-to-nearest or truncating adds) errs by at most (dim-1) * 2^-23 *
    sum|q_i e_i| <= dim * 2^-23 * |q| * |e| (Cauchy-Schwarz); a factor 2 of headroom
    covers the tensor core's internal accumulation order."""
    q = np.asarray(queries, dtype=np.float64)
    dim = q.shape[1]
    return 2.0 * dim * 2.0 ** -23 * np.linalg.norm(q, axis=1) * corpus_max_norm


def stage_ranking(scores: np.ndarray, ids: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """Top-(k+1) of one float64 score vector: (ids, scores), score desc / id asc."""
    return topk_rows(scores, ids, k + 1)


def staged_topk_margin(scores64: np.ndarray, k: int, n_stages: int, bound: np.ndarray,
                       id_offset: int = 0):
    """float64 scores [b, N] -> (ids [b,S,k], scores [b,S,k], ambiguous [b,S] bool,
    kth [b,S] float64 = the k-th best exact score of the stage).

    A stage is ambiguous when any adjacent gap among its top-(k+1) exact scores is
    <= 2 * bound (order or membership could flip under fp32 accumulation)."""
    b, n = scores64.shape
    ids_all = np.arange(n, dtype=np.int64) + id_offset
    out_ids = np.empty((b, n_stages, k), dtype=np.int64)
    out_sc = np.empty((b, n_stages, k))
    amb = np.zeros((b, n_stages), dtype=bool)
    kth = np.full((b, n_stages), -np.inf)
    for qi in range(b):
        for s in range(n_stages):
            bound_s = (n * (s + 1)) // n_stages
            r_ids, r_sc = stage_ranking(scores64[qi, :bound_s], ids_all[:bound_s], k)
            out_ids[qi, s], out_sc[qi, s] = r_ids[:k], r_sc[:k]
            fin = r_sc[np.isfinite(r_sc)]
            gaps = fin[:-1] - fin[1:]
            amb[qi, s] = bool((gaps <= 2.0 * bound[qi]).any())
            if len(fin) >= k:
                kth[qi, s] = fin[k - 1]
    return out_ids, out_sc, amb, kth


def check_topk_tolerant(got_ids, got_scores, exact_of, kth: float, bound: float) -> list[str]:
    """Problems (empty = ok) with one stage's GPU answer against exact float64 scores.

    got_ids/got_scores: the kernel's k ids (-1 = none) and fp32 scores;
    exact_of(id) -> float64 exact score of that id; kth = the stage's k-th best exact
    score.  Requirements: distinct ids; each fp32 score within `bound` of its exact
    score; each exact score >= kth - 2*bound (a legitimate top-k member); the list
    ordered by exact score up to 2*bound."""
    errs = []
    ids = [int(i) for i in got_ids if int(i) >= 0]
    if len(set(ids)) != len(ids):
        errs.append(f"duplicate ids {ids}")
    ex = []
    for i, sc in zip(got_ids, got_scores):
        if int(i) < 0:
            continue
        e = exact_of(int(i))
        ex.append(e)
        if abs(float(sc) - e) > bound:
            errs.append(f"id {int(i)}: fp32 score {float(sc)!r} vs exact {e!r} > bound {bound:.3g}")
        if e < kth - 2.0 * bound:
            errs.append(f"id {int(i)}: exact {e!r} below the k-th best {kth!r} - 2*bound")
    for a, c in zip(ex, ex[1:]):
        if c > a + 2.0 * bound:
            errs.append(f"order: exact {c!r} after {a!r}")
    return errs
