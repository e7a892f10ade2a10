"""GPU retrieval behind the reference's StageProvider seam.

ragsim asks ``stage_provider(req) -> StagedRetrieval`` at every arrival
(simulator.py:228, :366-372) and insists that the final stage equals the
request's ground-truth doc_sequence (:368-369).  ``GpuStageProvider``
answers from the tcgen05 staged top-k kernel (rcb_retrieval_topk): stage s is
the exact top-k over the first (s+1)/S of the scan order, so early stages
are genuine partial-search candidates that the DSP controller
(speculation.py:98-146) may speculate on.

``ShardedRetriever`` is the multi-GPU form: the corpus is split
in contiguous row shards, one per rank; a call all-gathers every rank's
queries, scans the local shard for all of them (passes of at most
``kernels.MAX_SCAN_QUERIES`` queries), all-gathers the per-shard staged lists
and merges them on device (rcb_topk_merge_shards, score desc / id asc).
Stage s globally = top-k over the union of every shard's first (s+1)/S rows
(oracle/topk_oracle.sharded_staged_topk).  With one rank it is a plain scan.

Because a ragsim run is trace-driven, the provider scans ahead: queries of up
to ``batch`` upcoming requests go through one retrieval call, and results are
served from that batch.  With several ranks every rank must call the
collectives in lockstep, so the provider precomputes its whole routed
sub-trace in rounds at construction (``prefetch``), padding short rounds.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels, synth
from ._ragsim import import_ragsim

import_ragsim()
from ragsim.speculation import StagedRetrieval  # noqa: E402

MAX_BATCH = 64


class ShardedRetriever:
    """Staged exact top-k over this rank's corpus shard, merged across ranks.

    corpus_shard  bf16 [N_shard, dim] on the device, global ids id_offset + row
    comm          paper_2404_12457_b200.dist.Dist (None = single rank)
    batch         queries per rank per call (calls pad to it: all ranks gather
                  equal-sized blocks)
    scan / merge  the kernels by default; tests on CPU inject the oracle to
                  exercise the collective logic without a GPU
    exchange      how the per-shard lists meet (world > 1): "p2p" = kernels.PeerExchange
                  (each rank pushes its lists into every peer's window over peer memory,
                  one merge kernel waits for all of them), "allgather" = two collective
                  all-gathers + the merge kernel; "auto" = p2p for device tensors with the
                  kernel merge, falling back to allgather if the IPC setup fails
    """

    def __init__(self, corpus_shard, id_offset: int, k: int, n_stages: int, comm=None, *,
                 batch: int = MAX_BATCH, pass_queries: int | None = None, scan=None,
                 merge=None, exchange: str = "auto") -> None:
        self.corpus = corpus_shard
        self.off = int(id_offset)
        self.k = k
        self.S = n_stages
        self.comm = comm
        self.world = comm.world if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.batch = batch
        nq = batch * self.world
        p = pass_queries or kernels.MAX_SCAN_QUERIES
        self.passes = [(a, min(nq, a + p)) for a in range(0, nq, p)]
        self._scan = scan
        self._merge = merge or kernels.topk_merge_shards
        dev = corpus_shard.device
        self.ws = {}
        if scan is None:
            for a, b in self.passes:
                if (b - a) not in self.ws:
                    self.ws[b - a] = kernels.RetrievalWorkspace(corpus_shard.shape[0], b - a, k,
                                                                n_stages, dev)
        self.ids = torch.empty((nq, n_stages, k), dtype=torch.int64, device=dev)
        self.sc = torch.empty((nq, n_stages, k), dtype=torch.float32, device=dev)
        self._qpad = torch.zeros((batch, corpus_shard.shape[1]), dtype=torch.bfloat16, device=dev)
        self.launches = 0
        self.bytes_per_scan = corpus_shard.shape[0] * corpus_shard.shape[1] * 2
        self.px = self.pq = None
        self.exchange = "allgather" if self.world == 1 else exchange
        if self.world > 1 and exchange in ("auto", "p2p"):
            if merge is None and dev.type == "cuda":
                try:
                    self.px = kernels.PeerExchange(comm, nq * n_stages * k,
                                                   lists=(nq, n_stages, k), device=dev)
                    qbytes = batch * corpus_shard.shape[1] * 2
                    if qbytes % 8 == 0:  # the queries too: no collective left in the loop
                        self.pq = kernels.PeerExchange(comm, qbytes // 8, device=dev)
                    self.exchange = "p2p" if self.pq is not None else "p2p lists"
                except RuntimeError as exc:  # CUDA IPC / peer mapping unavailable on this box
                    # (PeerExchange fails on every rank alike, so all ranks fall back together)
                    self.close()
                    if exchange == "p2p":
                        raise
                    self.exchange = f"allgather (peer exchange unavailable: {exc})"
            elif exchange == "p2p":
                raise ValueError("p2p exchange needs device tensors and the kernel merge")
            else:
                self.exchange = "allgather"

    def _scan_pass(self, q, a, b):
        if self._scan is not None:
            i, s = self._scan(self.corpus, q, self.k, self.S, self.off)
            self.ids[a:b].copy_(i)
            self.sc[a:b].copy_(s)
            return
        kernels.retrieval_topk(self.corpus, q, self.k, self.S, self.off, workspace=self.ws[b - a],
                               ids_out=self.ids[a:b], scores_out=self.sc[a:b])
        self.launches += 2

    def close(self) -> None:
        """Unmap the peers' exchange windows and free this rank's."""
        for px in (self.px, self.pq):
            if px is not None:
                px.close()
        self.px = self.pq = None

    def scan_all(self, allq: torch.Tensor) -> None:
        """Scan the local shard for a gathered [world*batch, dim] query block."""
        for a, b in self.passes:
            self._scan_pass(allq[a:b], a, b)

    def __call__(self, q_local: torch.Tensor, with_scores: bool = False):
        """q_local: [b <= batch, dim] bf16 -> ids int64 [b, S, k] (and fp32 scores)."""
        b = q_local.shape[0]
        if b > self.batch:
            raise ValueError(f"{b} queries > batch {self.batch}")
        if b < self.batch:
            self._qpad[:b].copy_(q_local)
            self._qpad[b:].zero_()
            q_local = self._qpad
        if self.world == 1:
            self.scan_all(q_local)
            return (self.ids[:b], self.sc[:b]) if with_scores else self.ids[:b]
        if self.pq is not None:  # over peer memory (ordering: kernels.PeerExchange)
            allq = self.pq.gather(q_local.contiguous())
        else:  # the collective also orders successive list exchanges
            allq = self.comm.all_gather(q_local).reshape(-1, q_local.shape[1])
        self.scan_all(allq)
        if self.px is not None:
            ids, sc = self.px.merge(self.ids, self.sc)
            self.launches += 3  # push, wait, merge
        else:
            gi = self.comm.all_gather(self.ids)  # [world, world*batch, S, k]
            gs = self.comm.all_gather(self.sc)
            ids, sc = self._merge(gi, gs)
            self.launches += 1
        r0 = self.rank * self.batch
        return (ids[r0:r0 + b], sc[r0:r0 + b]) if with_scores else ids[r0:r0 + b]

    def device_ms(self, q_block: torch.Tensor, reps: int = 20) -> float:
        """Device time of one local scan of a [world*batch, dim] query block (every pass,
        scan + merge kernels), replayed back to back from a CUDA graph (corpus >> L2)."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.scan_all(q_block)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(reps):
                    self.scan_all(q_block)
        torch.cuda.synchronize()
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps


class GpuStageProvider:
    """StageProvider for ragsim.run / TieredEngine.

    corpus      bf16 [N_shard, dim] on the GPU (row id = document id - id_offset)
    query_fn    req -> float array [dim] (the request's query embedding)
    stage_interval_ms  per-stage latency reported to the engine (the measured
                scan time in timed mode, the config knob in parity mode)
    comm, id_offset    corpus sharded across ranks; with
                comm.world > 1 the trace (this rank's routed requests) is required
                and scanned at construction in lockstep rounds
    """

    def __init__(self, corpus: torch.Tensor, query_fn, *, k: int, n_stages: int,
                 stage_interval_ms: float, trace=None, check_ground_truth: bool = True,
                 comm=None, id_offset: int = 0, batch: int = MAX_BATCH, retriever=None) -> None:
        self.corpus = corpus
        self.query_fn = query_fn
        self.k = k
        self.n_stages = n_stages
        self.stage_interval_ms = stage_interval_ms
        self.check = check_ground_truth
        self._cache: dict[int, np.ndarray] = {}
        self._upcoming = list(trace) if trace is not None else []
        self._pos = 0
        self.retriever = retriever or ShardedRetriever(corpus, id_offset, k, n_stages, comm,
                                                       batch=batch)
        self.batch = self.retriever.batch
        if self.retriever.world > 1:
            if trace is None:
                raise ValueError("a sharded provider needs the rank's trace (lockstep prefetch)")
            self.prefetch()

    @property
    def launches(self) -> int:
        return self.retriever.launches

    def _scan(self, reqs) -> None:
        dim = self.corpus.shape[1]
        q = np.stack([self.query_fn(r) for r in reqs]) if reqs else np.zeros((0, dim))
        q = torch.from_numpy(q.astype(np.float32)).to(self.corpus.device, torch.bfloat16)
        if q.shape[0] == 0:  # an idle rank still joins the round's collectives
            q = torch.zeros((1, dim), dtype=torch.bfloat16, device=self.corpus.device)
        ids = self.retriever(q).cpu().numpy()
        for r, row in zip(reqs, ids):
            self._cache[r.id] = row

    def prefetch(self) -> None:
        """Scan every upcoming request in rounds of ``batch``; all ranks run the same
        number of rounds (the longest routed trace decides)."""
        reqs = self._upcoming
        rounds = -(-len(reqs) // self.batch)
        comm = self.retriever.comm
        if comm is not None and comm.world > 1:
            rounds = int(comm.max(float(rounds)))
        for i in range(rounds):
            self._scan(reqs[i * self.batch:(i + 1) * self.batch])
        self._pos = len(reqs)

    def __call__(self, req) -> StagedRetrieval:
        row = self._cache.pop(req.id, None)
        if row is None:
            if self.retriever.world > 1:
                raise KeyError(f"request {req.id} is not in this rank's prefetched trace")
            # scan ahead over the known trace (or just this request)
            batch = [req]
            while self._pos < len(self._upcoming) and len(batch) < self.batch:
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


def synthetic_query_fn(seed: int = 0, dim: int = synth.EMB_DIM, kind: str = "real"):
    """Query embeddings built from each request's ground-truth documents, for
    the real (unit-norm bf16, the default) or the integer synthetic corpus."""
    if kind not in ("real", "int"):
        raise ValueError(f"kind must be real or int, not {kind!r}")

    def fn(req):
        rng = np.random.default_rng(np.random.SeedSequence([seed, 0x0BE7, req.id]))
        ids = np.asarray(req.doc_sequence, dtype=np.int64)
        if kind == "int":
            return synth.build_query_int(synth.int_rows(ids, dim, seed), jitter=1.0, rng=rng)
        return synth.build_query(synth.corpus_rows(ids, dim, seed), jitter=1.0, rng=rng)

    return fn
