"""ORACLE (test infrastructure + the bench's CPU arms only — never the product path).

The reference's CPU path for one hot-path step, used by ``bench.py --impl
reference`` and by the ``cpu_baseline`` leg of the GPU arm.  It must not load
libragcache_b200.so: nothing here imports the package's native modules
(``tests/test_ref_path.py`` checks the process maps).

* decisions: ragsim's own, UNMODIFIED ``KnowledgeTree`` (baseline/_ref) driven
  with ``SimulationEngine._admit`` / ``_commit``'s call sequences
  (simulator.py:481-534) — no TieredKnowledgeTree, no block pool, the
  reference's linear victim scan (tree.py:407-411);
* retrieval: numpy float64 exact staged top-k (oracle/topk_oracle.py) over the
  host-resident corpus;
* KV + attention: per request and layer, RoPE of the suffix queries/keys,
  the suffix K/V written into its node-aligned pages of a host KV pool, the
  request's pages gathered and fp32 prefix attention (oracle/attn_oracle.py),
  torch on all host threads.

A step serves the same batch as the GPU arm's step (same trace, same batching
and carry rule, so the tree reaches the same state); the TIMED part is a
bounded sample: the first ``n_sample`` requests of the step through the whole
path (their admit + commit, retrieval, every layer of KV write + gather +
attention).  The step's other requests are decided untimed so the tree
follows the GPU arm.  No extrapolation: value = sampled requests / time.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np
import torch

from oracle import attn_oracle, topk_oracle


class PlainTreeReplay:
    """ragsim.tree.KnowledgeTree with SimulationEngine._admit/_commit's sequences."""

    def __init__(self, gpu_tokens: int, host_tokens: int, sizes, profile, policy: str = "pgdsf"):
        from ragsim.policies import make_policy
        from ragsim.tree import KnowledgeTree

        self.tree = KnowledgeTree(gpu_tokens, host_tokens, policy=make_policy(policy))
        self.sizes = sizes
        self.profile = profile

    def admit(self, docs, prompt: int):
        """simulator.py:481-496: lookup -> pin -> evict_gpu -> load_to_gpu -> reserve_gpu.
        Returns (matched nodes, alpha, beta, promoted tokens); raises
        InsufficientEvictableCapacity exactly where the engine would requeue."""
        from ragsim.tree import InsufficientEvictableCapacity, Tier

        tree = self.tree
        match = tree.lookup(docs)
        miss = sum(self.sizes[d] for d in match.miss_docs)
        host_nodes = [n for n in match.matched_nodes if n.tier is Tier.HOST]
        need = sum(n.size for n in host_nodes) + miss + prompt
        tree.pin(match.matched_nodes)
        try:
            if tree.gpu_free < need:
                tree.evict_gpu(need - tree.gpu_free)
        except InsufficientEvictableCapacity:
            tree.unpin(match.matched_nodes)
            raise
        moved = tree.load_to_gpu(host_nodes)
        tree.reserve_gpu(miss + prompt)
        return list(match.matched_nodes), match.hit_tokens, miss + prompt, moved

    def commit(self, docs, adm) -> None:
        """simulator.py:516-530: release_gpu -> insert_path -> update_node x path -> unpin."""
        matched, alpha, beta, _ = adm
        tree = self.tree
        tree.release_gpu(beta)
        path = tree.insert_path(docs, [self.sizes[d] for d in docs])
        for i, node in enumerate(path):
            tree.update_node(node, i < len(matched), alpha, beta, self.profile)
        tree.unpin(matched)


def admit_step(admit, batch, R: int):
    """The GPU arm's batching rule (bench.run_ours / HotPath.admit_batch): requests left
    over from the previous step go first; admission stops at the first request that
    does not fit (InsufficientEvictableCapacity) and the rest carry over.
    Returns (admitted [(req, adm)], carry)."""
    from ragsim.tree import InsufficientEvictableCapacity

    cand, rest = batch[:R], batch[R:]
    out = []
    for r in cand:
        try:
            out.append((r, admit(r)))
        except InsufficientEvictableCapacity:
            break
    if not out:
        raise RuntimeError("a single request exceeds the GPU tier's evictable capacity")
    return out, cand[len(out):] + rest


class CpuKernels:
    """The CPU versions of the three hot-path kernels on a host-resident corpus and a
    host KV pool sized for the sample (node-aligned pages, like the device pool)."""

    def __init__(self, w, corpus_f32: np.ndarray, n_sample: int, max_blocks_per_req: int,
                 seed: int = 0):
        s = w.model
        self.w = w
        self.shape = s
        self.bt = w.block_tokens
        self.corpus64 = corpus_f32.astype(np.float64)  # the resident index (fp64 exact scores)
        g = torch.Generator().manual_seed(seed)
        nb = n_sample * max_blocks_per_req
        self.pool = torch.randn((nb, s.n_layers, 2, s.n_kv_heads, self.bt, s.head_dim),
                                generator=g).to(torch.bfloat16)
        self.max_blocks = max_blocks_per_req
        self.gen = g

    def retrieval(self, queries: np.ndarray):
        q = np.asarray(queries, dtype=np.float64)
        return topk_oracle.staged_topk_from_scores(q @ self.corpus64.T, self.w.k, self.w.n_stages)

    def table(self, slot: int, matched_sizes, suffix_sizes):
        """Node-aligned block table of one sampled request in its private pool range."""
        blocks, valid = [], []
        b = slot * self.max_blocks
        for n in list(matched_sizes) + list(suffix_sizes):
            for j in range(-(-n // self.bt)):
                blocks.append(b)
                valid.append(min(self.bt, n - j * self.bt))
                b += 1
        if b > (slot + 1) * self.max_blocks:
            raise ValueError("sample request exceeds its pool range")
        return blocks, valid

    def prefill(self, alpha: int, beta: int, blocks, valid, n_prefix_blocks: int,
                q_raw: torch.Tensor, kv_raw: torch.Tensor) -> torch.Tensor:
        """Every layer: RoPE(q, k) of the suffix, K/V written into the suffix pages, pages
        gathered, fp32 prefix attention.  q_raw [beta, Hq, d], kv_raw [2, beta, Hkv, d]."""
        s = self.shape
        pos = torch.arange(alpha, alpha + beta)
        slots = []
        for b, v in zip(blocks[n_prefix_blocks:], valid[n_prefix_blocks:]):
            slots.extend(b * self.bt + o for o in range(v))
        slots = torch.tensor(slots)
        blk, off = slots // self.bt, slots % self.bt
        reqs = [(beta, alpha, blocks, valid)]
        out = None
        for layer in range(s.n_layers):
            q = attn_oracle.apply_rope(q_raw, pos, s.rope_theta)
            k = attn_oracle.apply_rope(kv_raw[0], pos, s.rope_theta).to(torch.bfloat16)
            # pool[b, layer, kv, h, off, :] = suffix token t's K / V (paged write)
            self.pool[blk, layer, 0, :, off, :] = k
            self.pool[blk, layer, 1, :, off, :] = kv_raw[1]
            out = attn_oracle.prefix_prefill(q, self.pool, reqs, layer)
        return out


def cpu_gather_gbs(block_bytes: int, n_blocks: int = 64, n_pick: int = 32) -> dict:
    """CPU KV-gather comparator: index_select of n_pick random blocks of a
    host pool into a contiguous buffer on all host threads; bytes = read + write."""
    nb = max(n_blocks, n_pick)
    pool = torch.randint(0, 255, (nb, block_bytes), dtype=torch.uint8)
    idx = torch.from_numpy(np.random.default_rng(0).permutation(nb)[:n_pick].copy())
    out = torch.empty((n_pick, block_bytes), dtype=torch.uint8)
    torch.index_select(pool, 0, idx, out=out)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        torch.index_select(pool, 0, idx, out=out)
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[len(ts) // 2]
    return {"gbs": round(2 * n_pick * block_bytes / t / 1e9, 2), "blocks": n_pick,
            "block_bytes": block_bytes, "threads": torch.get_num_threads(),
            "how": "torch.index_select of random KV blocks of a host pool, median of 5, "
                   "read + write bytes"}


def host_decision_us(w, profile_path: str | None, n_requests: int = 1500, seed: int = 0) -> dict:
    """ragsim's own engine (ragsim.simulator.run, decisions + virtual clock, unmodified) on
    this workload's stream: host decision time per request on one core."""
    from ragsim.config import RunConfig
    from ragsim.simulator import run

    from paper_2404_12457_b200.workloads import make_stream

    trace, sizes = make_stream(w, n_requests, rate=2.0, seed=seed)
    cfg = RunConfig(gpu_capacity_tokens=w.gpu_capacity_tokens,
                    host_capacity_tokens=w.host_capacity_tokens, k=w.k, seed=seed,
                    kv_bytes_per_token=float(w.model.kv_bytes_per_token),
                    **({"profile_path": profile_path} if profile_path else {}))
    t0 = time.process_time()
    rep = run(cfg, trace, sizes)
    dt = time.process_time() - t0
    return {"us_per_request": round(dt / len(trace) * 1e6, 1), "requests": len(trace),
            "cores": 1, "doc_hit_rate": round(rep.aggregates()["doc_hit_rate"], 4),
            "how": "ragsim.simulator.run (unmodified engine: tree, PGDSF, queue, virtual "
                   "clock), process CPU time / requests"}


def run_cpu_path(w, steps, sizes, profile, *, R: int, n_warm: int, n_steps: int,
                 n_sample: int = 2, seed: int = 0) -> dict:
    """Replay the GPU arm's batches on the plain tree: n_warm untimed steps, then n_steps
    steps whose first n_sample requests are timed through the whole CPU path."""
    from paper_2404_12457_b200 import synth

    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    plain = PlainTreeReplay(w.gpu_capacity_tokens, w.host_capacity_tokens, sizes, profile)
    shape = w.model
    max_doc = max(sizes.values())
    max_blocks = w.k * (-(-max_doc // w.block_tokens)) + -(-w.prompt_tokens // w.block_tokens) + 2
    t0 = time.perf_counter()
    corpus = synth.corpus_f32(w.num_docs, seed=w.seed)
    kern = CpuKernels(w, corpus, n_sample, max_blocks, seed=seed)
    setup_s = time.perf_counter() - t0
    admit = lambda r: plain.admit(r.doc_sequence, r.prompt_tokens)  # noqa: E731
    carry = []
    step_s, served, hits, docs_total, exact = [], 0, 0, 0, True
    g = torch.Generator().manual_seed(seed + 1)
    for i in range(n_warm + n_steps):
        batch = carry + list(steps[i])
        timed = i >= n_warm
        if not timed:
            adm, carry = admit_step(admit, batch, R)
            for r, a in adm:
                plain.commit(r.doc_sequence, a)
            continue
        # the step's first n_sample requests through the whole path (timed)
        head = batch[:min(n_sample, R)]
        qs = synth.build_queries(lambda ids: corpus[ids], [r.doc_sequence for r in head],
                                 seed=head[0].id)
        inputs = []
        for r in head:  # suffix activations (the model projections' outputs), untimed
            beta_max = sum(sizes[d] for d in r.doc_sequence) + r.prompt_tokens
            inputs.append((torch.randn((beta_max, shape.n_q_heads, shape.head_dim), generator=g),
                           torch.randn((2, beta_max, shape.n_kv_heads, shape.head_dim),
                                       generator=g).to(torch.bfloat16)))
        from ragsim.tree import InsufficientEvictableCapacity

        t_a = time.perf_counter()
        ids, _ = kern.retrieval(qs)
        exact &= [tuple(int(x) for x in row) for row in ids[:, -1]] == \
            [tuple(r.doc_sequence) for r in head]
        adm_head = []
        for r in head:
            try:
                adm_head.append((r, admit(r)))
            except InsufficientEvictableCapacity:
                break
        t_timed = time.perf_counter() - t_a
        # the rest of the step's admissions (untimed), in the GPU arm's order: every
        # admission of the step happens before any commit (HotPath.admit_batch, then commit)
        rest_adm = []
        if len(adm_head) == len(head):
            for r in batch[len(head):R]:
                try:
                    rest_adm.append((r, admit(r)))
                except InsufficientEvictableCapacity:
                    break
        if not adm_head and not rest_adm:
            raise RuntimeError("a single request exceeds the GPU tier's evictable capacity")
        carry = batch[len(adm_head) + len(rest_adm):]
        t_a = time.perf_counter()
        for slot, (r, a) in enumerate(adm_head):
            matched, alpha, beta, _ = a
            miss = list(r.doc_sequence[len(matched):])
            blocks, valid = kern.table(slot, [n.size for n in matched],
                                       [sizes[d] for d in miss] + [r.prompt_tokens])
            n_pre = sum(-(-n.size // w.block_tokens) for n in matched)
            q_raw, kv_raw = inputs[slot]
            kern.prefill(alpha, beta, blocks, valid, n_pre, q_raw[:beta], kv_raw[:, :beta])
        for r, a in adm_head:
            plain.commit(r.doc_sequence, a)
        step_s.append(t_timed + time.perf_counter() - t_a)
        for r, a in rest_adm:
            plain.commit(r.doc_sequence, a)
        served += len(adm_head)
        hits += sum(len(a[0]) for _, a in adm_head)
        docs_total += sum(len(r.doc_sequence) for r, _ in adm_head)
    total = sum(step_s)
    return {"value": served / total if total > 0 else 0.0, "unit": "req/s",
            "ms_per_step": 1e3 * total / max(1, len(step_s)), "steps": len(step_s),
            "served": served, "cores": threads, "setup_s": round(setup_s, 2),
            "doc_hit_rate": round(hits / max(1, docs_total), 4),
            "retrieval_matches_ground_truth": bool(exact),
            "sample": (f"per step: the first {n_sample} of the step's {R} requests through the "
                       f"reference CPU path, all timed, no extrapolation: ragsim's unmodified "
                       f"KnowledgeTree admit/commit (linear victim scan), numpy float64 exact "
                       f"staged top-{w.k} over {w.num_docs} docs, and for all "
                       f"{shape.n_layers} layers RoPE + paged K/V write + page gather + fp32 "
                       f"prefix attention (torch, {threads} threads); the step's other "
                       f"requests decided untimed so the tree follows the GPU arm")}
