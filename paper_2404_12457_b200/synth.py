"""Synthetic inputs for the hot path: embedding corpus and queries.

Two corpora, both reproducible row by row from a counter hash of
(seed, row, column), so any shard is generated on its own, on the CPU or on
the GPU, with identical bytes:

* the REAL corpus (the product/bench data): each row is an
  Irwin-Hall(4) integer vector (sum of four hash bytes minus 510, ~N(0, 148^2))
  scaled to unit L2 norm and stored bf16, i.e. N(0,1)/sqrt(768)-like,
  L2-normalised bf16 embeddings.  The normalisation is made bit-reproducible:
  the sum of squares is an exact int64, 1/sqrt(.) and the product are single
  correctly rounded fp64 operations, then fp64 -> fp32 -> bf16 round to
  nearest even on both sides.  Inner products are NOT exact in fp32, so parity
  of retrieved ids is margin-aware (oracle/topk_oracle.py).
* the INTEGER corpus (kernel tests only): integer-valued bf16 in [-8, 8];
  every inner product with an integer query |q| <= 240 is an integer < 2^24,
  exact in fp32 under any accumulation order, which pins the kernel's
  selection logic (ties included) bit for bit.

A request's query is built from its ground-truth documents (the trace's
doc_sequence, ragsim workload.py:124-148): solve the k x k Gram system so the
targets score t_i = 1 + 0.1*(k-1-i) (jittered 1%) in relevance order,
normalise (real) or scale to |q| <= 240 and round (integer).
"""

from __future__ import annotations

import numpy as np

EMB_DIM = 768
EMB_MAX = 8
Q_MAX = 240


_M1, _M2, _M3, _MIX = 0x27D4EB2D, 0x165667B1, 0x3C6EF372, 0x045D9F3B
_MASK = 0xFFFFFFFF
_IH_BIAS = 510  # Irwin-Hall(4) of bytes: mean 4 * 127.5


def _hash32_np(x: np.ndarray) -> np.ndarray:
    # every product stays below 2^63 (32-bit value x 27-bit constant)
    x = ((x ^ (x >> 16)) * _MIX) & _MASK
    x = ((x ^ (x >> 16)) * _MIX) & _MASK
    return x ^ (x >> 16)


def _cell_hash_np(rows: np.ndarray, dim: int, seed: int) -> np.ndarray:
    r = np.asarray(rows, dtype=np.int64)[:, None]
    c = np.arange(dim, dtype=np.int64)[None, :]
    return _hash32_np((r * _M1 + c * _M2 + (seed & 0xFFFF) * _M3) & _MASK)


def to_bf16_f32(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16 (ties to even) and return it as float32 (finite inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


# ---------------------------------------------------------------------- real corpus
def _normalise_rows_np(u: np.ndarray) -> np.ndarray:
    ss = (u.astype(np.int64) ** 2).sum(axis=1, keepdims=True)  # exact
    inv = 1.0 / np.sqrt(ss.astype(np.float64))
    return to_bf16_f32((u.astype(np.float64) * inv).astype(np.float32))


def corpus_rows(rows: np.ndarray, dim: int = EMB_DIM, seed: int = 0) -> np.ndarray:
    """float32 [len(rows), dim] holding bf16 values: unit-norm Irwin-Hall rows."""
    h = _cell_hash_np(rows, dim, seed)
    u = (h & 0xFF) + ((h >> 8) & 0xFF) + ((h >> 16) & 0xFF) + ((h >> 24) & 0xFF) - _IH_BIAS
    return _normalise_rows_np(u)


def corpus_f32(n_rows: int, dim: int = EMB_DIM, seed: int = 0, row_offset: int = 0) -> np.ndarray:
    """Rows [row_offset, row_offset + n_rows) of the real corpus (float32 holding bf16)."""
    out = np.empty((n_rows, dim), dtype=np.float32)
    step = 1 << 15
    for lo in range(0, n_rows, step):
        hi = min(n_rows, lo + step)
        out[lo:hi] = corpus_rows(np.arange(row_offset + lo, row_offset + hi), dim, seed)
    return out


def corpus_device(n_rows: int, dim: int = EMB_DIM, seed: int = 0, row_offset: int = 0,
                  device="cuda", chunk: int = 1 << 16):
    """Same rows as corpus_f32, generated on the device: bf16 [n_rows, dim]."""
    import torch

    out = torch.empty((n_rows, dim), dtype=torch.bfloat16, device=device)
    c = torch.arange(dim, dtype=torch.int64, device=device)[None, :]
    for lo in range(0, n_rows, chunk):
        hi = min(n_rows, lo + chunk)
        r = torch.arange(row_offset + lo, row_offset + hi, dtype=torch.int64, device=device)[:, None]
        x = (r * _M1 + c * _M2 + (seed & 0xFFFF) * _M3) & _MASK
        x = ((x ^ (x >> 16)) * _MIX) & _MASK
        x = ((x ^ (x >> 16)) * _MIX) & _MASK
        h = x ^ (x >> 16)
        u = (h & 0xFF) + ((h >> 8) & 0xFF) + ((h >> 16) & 0xFF) + ((h >> 24) & 0xFF) - _IH_BIAS
        ss = (u * u).sum(dim=1, keepdim=True)  # exact int64
        inv = torch.reciprocal(torch.sqrt(ss.to(torch.float64)))
        out[lo:hi] = (u.to(torch.float64) * inv).to(torch.float32).to(torch.bfloat16)
    return out


def target_scores(k: int) -> np.ndarray:
    return np.array([1.0 + 0.1 * (k - 1 - i) for i in range(k)], dtype=np.float64)


def _solve_targets(e: np.ndarray, jitter: float, rng) -> np.ndarray:
    k = e.shape[0]
    t = target_scores(k)
    if jitter and rng is not None:
        t = t * (1.0 + jitter * rng.standard_normal(k) * 0.01)
        t = np.sort(t)[::-1]
    gram = e @ e.T
    a = np.linalg.solve(gram + 1e-9 * np.eye(k), t)
    return a @ e


def build_query(target_rows: np.ndarray, jitter: float = 0.0,
                rng: np.random.Generator | None = None) -> np.ndarray:
    """Unit-norm query (float32 holding bf16) whose scores against the k target rows are
    descending in the given order, ~0.07 apart at k=2 (random rows score ~N(0, 1/768))."""
    q = _solve_targets(target_rows.astype(np.float64), jitter, rng)
    q /= max(1e-12, float(np.linalg.norm(q)))
    return to_bf16_f32(q.astype(np.float32))


def build_queries(corpus_rows_fn, doc_sequences, seed: int = 0) -> np.ndarray:
    """[b, dim] float32 (bf16 values) real queries; corpus_rows_fn(ids) -> those rows."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x0BE7]))
    out = []
    for docs in doc_sequences:
        rows = corpus_rows_fn(np.asarray(docs, dtype=np.int64))
        out.append(build_query(rows, jitter=1.0, rng=rng))
    return np.stack(out) if out else np.zeros((0, EMB_DIM), dtype=np.float32)


# ---------------------------------------------------------------------- integer corpus
def int_rows(rows: np.ndarray, dim: int = EMB_DIM, seed: int = 0) -> np.ndarray:
    """int8 [len(rows), dim] in [-EMB_MAX, EMB_MAX]."""
    return (_cell_hash_np(rows, dim, seed) % (2 * EMB_MAX + 1) - EMB_MAX).astype(np.int8)


def corpus_int(n_rows: int, dim: int = EMB_DIM, seed: int = 0, row_offset: int = 0) -> np.ndarray:
    """Rows [row_offset, row_offset + n_rows) of the integer corpus."""
    out = np.empty((n_rows, dim), dtype=np.int8)
    step = 1 << 16
    for lo in range(0, n_rows, step):
        hi = min(n_rows, lo + step)
        out[lo:hi] = int_rows(np.arange(row_offset + lo, row_offset + hi), dim, seed)
    return out


def build_query_int(target_rows: np.ndarray, jitter: float = 0.0,
                    rng: np.random.Generator | None = None) -> np.ndarray:
    """Integer query (float64 holding ints, |q| <= Q_MAX) for the integer corpus."""
    q = _solve_targets(target_rows.astype(np.float64), jitter, rng)
    q *= Q_MAX / max(1e-12, np.abs(q).max())
    return np.rint(q)


def build_queries_int(corpus_rows_fn, doc_sequences, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x0BE7]))
    out = []
    for docs in doc_sequences:
        rows = corpus_rows_fn(np.asarray(docs, dtype=np.int64))
        out.append(build_query_int(rows, jitter=1.0, rng=rng))
    return np.stack(out) if out else np.zeros((0, EMB_DIM))
