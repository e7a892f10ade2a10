"""Generate the block-pool golden fixtures FROM THE REFERENCE ITSELF.

Runs the unmodified ragsim engine (imported from /root/reference/pkg/src or
baseline/_ref) on desk-scale recipes modelled on the reference's acceptance
suite (pkg/tests/test_acceptance.py:33-41, C7 :334-361, C8 :364-383), with
the tier-transition hooks of paper_2404_12457_b200.cache feeding the Python
block oracle.  Records, per recipe:
  * the reference's own report (aggregates, per-request CSV) with and without
    the hooks — they must be identical;
  * the full pool event stream and every admission's block table;
  * final per-node GPU/host block lists and the tree's token accounting.

    python tests/golden/make_golden.py        # rewrites tests/golden/*.json.gz
"""

import dataclasses
import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.block_oracle import BlockOracle, EventRecorder  # noqa: E402
from paper_2404_12457_b200 import cache  # noqa: E402
from ragsim.config import RunConfig  # noqa: E402
from ragsim.simulator import run  # noqa: E402
from ragsim.tree import Tier  # noqa: E402
from ragsim.workload import PRESETS, TraceSpec, generate_corpus, generate_trace  # noqa: E402

MIB = 1024.0 * 1024.0
DESK = dict(gpu_capacity_tokens=10240, profile_base_ms=20.0, profile_per_token_ms=0.015,
            profile_attention_ms=1e-5, kv_bytes_per_token=0.5 * MIB)

RECIPES = {
    # C8-like: swaps, swap-ins, host frees (pkg/tests/test_acceptance.py:364-383)
    "desk_c8": dict(seed=3, duration_s=300.0, rate=0.6, pool=400,
                    cfg=dict(host_capacity_tokens=24576, dsp=True, stage_count=4,
                             stage_interval_ms=25.0, convergence_stage=2, seed=3)),
    # tight host tier: dropped evictions + _drop_subtree, LRU policy, no DSP
    "desk_drop_lru": dict(seed=5, duration_s=200.0, rate=0.8, pool=300,
                          cfg=dict(host_capacity_tokens=3000, policy="lru", seed=5)),
    # C7-like speculation-heavy run (pkg/tests/test_acceptance.py:334-361)
    "desk_c7_dsp": dict(seed=0, duration_s=250.0, rate=0.25, pool=300,
                        cfg=dict(host_capacity_tokens=32768, stage_count=4, stage_interval_ms=50.0,
                                 convergence_stage=2, prefill_chunk_ms=25.0, dsp=True, seed=0)),
}
BLOCK_TOKENS = 16


def desk_trace(seed, duration_s, rate, pool):
    corpus_spec = dataclasses.replace(PRESETS["mmlu"], num_docs=1500)
    rng = np.random.default_rng(np.random.SeedSequence([seed]))
    corpus = generate_corpus(corpus_spec, rng)
    spec = TraceSpec(duration_s=duration_s, arrival_rate=rate, seed=seed, query_pool=pool,
                     query_zipf_s=1.1, drift_interval_s=300.0, drift_fraction=0.3)
    return generate_trace(corpus, spec, rng), corpus.size_map()


def pool_geometry(cfg: RunConfig, sizes) -> tuple[int, int]:
    """Blocks for the tree's token capacity plus one tail block per resident node
     plus one in-flight generation's segments."""
    min_doc = min(sizes.values())
    g = -(-cfg.gpu_capacity_tokens // BLOCK_TOKENS) + cfg.gpu_capacity_tokens // min_doc + 8
    h = -(-cfg.host_capacity_tokens // BLOCK_TOKENS) + cfg.host_capacity_tokens // min_doc + 8
    return g, h


def make(name, r):
    trace, sizes = desk_trace(r["seed"], r["duration_s"], r["rate"], r["pool"])
    cfg = RunConfig(validate=True, **{**DESK, **r["cfg"]})
    plain = run(cfg, trace, sizes)
    ng, nh = pool_geometry(cfg, sizes)
    rec = EventRecorder(BlockOracle(ng, nh, BLOCK_TOKENS))
    report, engine = cache.run_tiered(cfg, trace, sizes, pool=rec, record_tables=True)
    assert report.to_json(cfg) == plain.to_json(cfg)
    assert report.per_request_csv() == plain.per_request_csv()
    nodes = {}
    for node in engine.tree.nodes():
        nodes[str(node.serial)] = {
            "path": [],
            "tier": node.tier.value,
            "tokens": node.size,
            "gpu": rec.inner.node_blocks(node.serial, 0),
            "host": rec.inner.node_blocks(node.serial, 1),
        }
        n, path = node, []
        while n is not None and n.parent is not None:
            path.append(n.doc)
            n = n.parent
        nodes[str(node.serial)]["path"] = path[::-1]
    gpu_tokens = sum(v["tokens"] for v in nodes.values() if v["tier"] == Tier.GPU.value)
    host_tokens = sum(v["tokens"] for v in nodes.values() if v["host"])
    assert gpu_tokens == engine.tree.gpu.used and host_tokens == engine.tree.host.used
    return {
        "recipe": {k: v for k, v in r.items()},
        "config": {f.name: getattr(cfg, f.name) for f in dataclasses.fields(cfg)},
        "block_tokens": BLOCK_TOKENS,
        "num_gpu_blocks": ng,
        "num_host_blocks": nh,
        "aggregates": report.aggregates(),
        "events": rec.events,
        "nodes": nodes,
    }


if __name__ == "__main__":
    for name, r in RECIPES.items():
        g = make(name, r)
        path = os.path.join(HERE, f"{name}.json.gz")
        with gzip.open(path, "wt") as fp:
            json.dump(g, fp, sort_keys=True, default=list)
        kinds = {}
        for ev in g["events"]:
            kinds[ev[0]] = kinds.get(ev[0], 0) + 1
        print(name, os.path.getsize(path), "bytes", kinds,
              {k: g["aggregates"][k] for k in ("swap_outs", "dropped_evictions", "host_evictions",
                                               "gpu_evictions", "doc_hit_rate")})
