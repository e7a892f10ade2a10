"""GPU retrieval behind the reference's StageProvider seam.

ragsim asks ``stage_provider(req) -> StagedRetrieval`` at every arrival
(simulator.py:228, :366-372) and insists that the final stage equals the
request's ground-truth doc_sequence (:368-369).  ``GpuStageProvider``
answers from the tcgen05 staged top-k kernel (rcb_retrieval_topk): stage s is
the exact top-k over the first (s+1)/S of the scan order, so early stages
are genuine partial-search candidates that the DSP controller
(speculation.py:98-146) may speculate on.

Because a ragsim run is trace-driven, the provider scans ahead: queries of up
to 64 upcoming requests go through one kernel launch, and results are served
from that batch (one launch per 64 arrivals instead of one per arrival).
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels, synth
from ._ragsim import import_ragsim

import_ragsim()
from ragsim.speculation import StagedRetrieval  # noqa: E402

MAX_BATCH = 64


class GpuStageProvider:
    """StageProvider for ragsim.run / TieredEngine.

    corpus      bf16 [N, dim] on the GPU (row id = document id)
    query_fn    req -> float array [dim] (the request's query embedding)
    stage_interval_ms  per-stage latency reported to the engine (the measured
                scan time in timed mode, the config knob in parity mode)
    """

    def __init__(self, corpus: torch.Tensor, query_fn, *, k: int, n_stages: int,
                 stage_interval_ms: float, trace=None, check_ground_truth: bool = True) -> None:
        self.corpus = corpus
        self.query_fn = query_fn
        self.k = k
        self.n_stages = n_stages
        self.stage_interval_ms = stage_interval_ms
        self.check = check_ground_truth
        self._cache: dict[int, np.ndarray] = {}
        self._upcoming = list(trace) if trace is not None else []
        self._pos = 0
        self.launches = 0
        self._ws = {}

    def _scan(self, reqs) -> None:
        q = torch.from_numpy(np.stack([self.query_fn(r) for r in reqs]).astype(np.float32))
        q = q.to(self.corpus.device, torch.bfloat16)
        b = q.shape[0]
        ws = self._ws.get(b)
        if ws is None:
            ws = self._ws[b] = kernels.RetrievalWorkspace(self.corpus.shape[0], b, self.k,
                                                          self.n_stages, self.corpus.device)
        ids, _ = kernels.retrieval_topk(self.corpus, q, self.k, self.n_stages, workspace=ws)
        self.launches += 2
        ids = ids.cpu().numpy()
        for r, row in zip(reqs, ids):
            self._cache[r.id] = row

    def __call__(self, req) -> StagedRetrieval:
        row = self._cache.pop(req.id, None)
        if row is None:
            # scan ahead over the known trace (or just this request)
            batch = [req]
            while self._pos < len(self._upcoming) and len(batch) < MAX_BATCH:
                nxt = self._upcoming[self._pos]
                self._pos += 1
                if nxt.id != req.id and nxt.id not in self._cache:
                    batch.append(nxt)
            self._scan(batch)
            row = self._cache.pop(req.id)
        staged = StagedRetrieval(tuple(tuple(int(x) for x in st) for st in row),
                                 self.stage_interval_ms)
        if self.check and staged.final_docs != tuple(req.doc_sequence):
            raise AssertionError(f"request {req.id}: retrieved {staged.final_docs}, "
                                 f"ground truth {tuple(req.doc_sequence)}")
        return staged


def synthetic_query_fn(seed: int = 0, dim: int = synth.EMB_DIM):
    """Query embeddings built from each request's ground-truth documents."""
    def fn(req):
        rng = np.random.default_rng(np.random.SeedSequence([seed, 0x0BE7, req.id]))
        rows = synth.corpus_rows(np.asarray(req.doc_sequence, dtype=np.int64), dim, seed)
        return synth.build_query(rows, jitter=1.0, rng=rng)

    return fn
