"""Model shapes and the BASELINE.json workloads (synthetic, reproducible).

Only the attention-relevant geometry of each model matters on the hot path
(KV bytes/token, query/kv heads, head dim): kvB = 2 * L * H_kv * d_h * 2
bytes (PAPER.md:802-807 gives 0.125 MiB for Mistral-7B /
Mixtral, 0.5 MiB for LLaMA2-7B).  Request streams come from the reference's
own generators (ragsim workload.py:114-195) seeded with SeedSequence([seed])
exactly as its CLI does (cli.py:169), so the GPU path and the CPU reference
see identical synthetic streams.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    rope_theta: float = 10000.0

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2

    @property
    def qkv_width(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim


SHAPES = {
    "tiny": ModelShape("tiny", 2, 4, 4, 64),
    "mistral-7b": ModelShape("mistral-7b", 32, 32, 8, 128),
    "llama2-7b": ModelShape("llama2-7b", 32, 32, 32, 128),
    "llama2-13b": ModelShape("llama2-13b", 40, 40, 40, 128),
    "mixtral-8x7b": ModelShape("mixtral-8x7b", 32, 32, 8, 128, 1e6),
}


@dataclass(frozen=True)
class Workload:
    name: str
    shape: str
    num_docs: int
    doc_tokens_mean: float
    doc_tokens_sigma: float
    zipf_s: float
    k: int
    prompt_tokens: int
    gpu_capacity_tokens: int
    host_capacity_tokens: int
    block_tokens: int
    n_stages: int = 4
    batch: int = 64  # requests per hot-path step (per GPU)
    query_pool: int | None = None
    query_zipf_s: float = 0.0
    seed: int = 0

    @property
    def model(self) -> ModelShape:
        return SHAPES[self.shape]


WORKLOADS = {
    # configs[0]: the CPU reference's own desk case (tiny LLaMA-style, 1K docs, top-2, PGDSF)
    "tiny-1k": Workload("tiny-1k", "tiny", 1000, 600.0, 1.5, 0.97, 2, 32, 10240, 32768, 16,
                        batch=32, query_pool=300, query_zipf_s=1.1),
    # configs[1]: Mistral-7B shape, 100K docs x 512 tokens, top-2, Zipf popularity, one B200.
    # GPU tier = (HBM - 14.5 GB weights - workspace) / 128 KiB ~ 1.1M tokens;
    # single tier (host 0: evicted nodes are dropped) — configs[2] exercises the host tier.
    "mistral7b-100k": Workload("mistral7b-100k", "mistral-7b", 100_000, 512.0, 0.0, 0.97, 2, 32,
                               1_100_000, 0, 64),
    # configs[1] shape with MMLU-like repeated questions (query pool, Zipf 1.1 over
    # questions, as the reference's desk recipe pkg/tests/test_acceptance.py:33-41):
    # the hit-rate axis of the TTFT curve
    "mistral7b-100k-qpool": Workload("mistral7b-100k-qpool", "mistral-7b", 100_000, 512.0, 0.0,
                                     0.97, 2, 32, 1_100_000, 0, 64, query_pool=20_000,
                                     query_zipf_s=1.1),
    # configs[2]: LLaMA2-7B shape, top-5, two-tier cache under memory pressure
    "llama2-7b-top5": Workload("llama2-7b-top5", "llama2-7b", 100_000, 512.0, 0.0, 0.97, 5, 32,
                               40_000, 160_000, 64, batch=12),
    # configs[2] with repeated questions (query pool, Zipf 1.1 over questions): the
    # host tier then serves real hits, which the layer-pipelined swap-in targets
    "llama2-7b-top5-qpool": Workload("llama2-7b-top5-qpool", "llama2-7b", 100_000, 512.0, 0.0,
                                     0.97, 5, 32, 40_000, 160_000, 64, batch=12,
                                     query_pool=500, query_zipf_s=1.1),
    # configs[3]: LLaMA2-13B shape, 10M-doc corpus sharded over the GPUs, DSP stages
    # (kvB = 800 KiB/token: a 120K-token tier is 98 GB next to 26 GB of weights)
    "llama2-13b-10m": Workload("llama2-13b-10m", "llama2-13b", 10_000_000, 512.0, 0.0, 0.97, 2,
                               32, 120_000, 0, 64, batch=32),
    # configs[4]: Mixtral-8x7B shape, Poisson arrivals, reordering, DP replicas
    "mixtral-poisson": Workload("mixtral-poisson", "mixtral-8x7b", 100_000, 512.0, 0.0, 0.97, 2,
                                32, 400_000, 100_000, 64),
}


def make_stream(w: Workload, n_requests: int, rate: float = 1.0, seed: int | None = None):
    """(trace, sizes) from the reference's generators (identical synthetic stream)."""
    from ._ragsim import import_ragsim

    import_ragsim()
    from ragsim.workload import CorpusSpec, TraceSpec, generate_corpus, generate_trace

    seed = w.seed if seed is None else seed
    spec = CorpusSpec(num_docs=w.num_docs, length_mean=w.doc_tokens_mean,
                      length_sigma=w.doc_tokens_sigma, zipf_s=w.zipf_s)
    rng = np.random.default_rng(np.random.SeedSequence([seed]))
    corpus = generate_corpus(spec, rng)
    duration = max(1.0, n_requests / rate * 1.02 + 5.0)
    tspec = TraceSpec(duration_s=duration, arrival_rate=rate, k=w.k,
                      prompt_tokens=w.prompt_tokens, query_pool=w.query_pool,
                      query_zipf_s=w.query_zipf_s, seed=seed)
    trace = generate_trace(corpus, tspec, rng)
    while len(trace) < n_requests:  # Poisson count fell short: extend the horizon
        duration *= 1.2
        rng = np.random.default_rng(np.random.SeedSequence([seed]))
        corpus = generate_corpus(spec, rng)
        trace = generate_trace(corpus, dataclasses.replace(tspec, duration_s=duration), rng)
    return trace[:n_requests], corpus.size_map()


def pool_blocks(capacity_tokens: int, block_tokens: int, doc_sizes,
                inflight_segments: int) -> int:
    """Blocks covering a token capacity: ceil(cap/B) + one tail block per resident node
    whenever any document (node) size is not a multiple of B (at most
    cap // smallest-doc nodes fit) + in-flight generation segments (+8 slack).
    ``doc_sizes``: the corpus sizes (iterable or dict values)."""
    if capacity_tokens <= 0:
        return 0
    sizes = list(doc_sizes)
    ragged = any(int(s) % block_tokens for s in sizes)
    tails = capacity_tokens // max(1, min(sizes)) if ragged else 0
    return -(-capacity_tokens // block_tokens) + tails + inflight_segments + 8
