"""Bundle formats for real runs: embeddings file next to ragsim's
corpus.csv / trace.jsonl (workload.py:203-259), and the extended run report."""

import json
import os

import numpy as np
import pytest
import torch

from paper_2404_12457_b200 import formats, synth
from paper_2404_12457_b200._ragsim import ragsim_available


def test_embeddings_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((37, 128)).astype(np.float32) * 3
    p = str(tmp_path / "e.rcbemb")
    formats.write_embeddings(p, torch.from_numpy(x).to(torch.bfloat16))
    assert formats.read_header(p) == (37, 128)
    got = np.asarray(formats.read_embeddings(p))
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref)
    # float input is rounded like torch's bf16 cast (round to nearest even)
    p2 = str(tmp_path / "f.rcbemb")
    formats.write_embeddings(p2, x)
    assert np.array_equal(np.asarray(formats.read_embeddings(p2)), ref)
    # a row slice reads only those rows
    assert np.array_equal(np.asarray(formats.read_embeddings(p, slice(5, 9))), ref[5:9])


def test_header_validation(tmp_path):
    p = str(tmp_path / "e.rcbemb")
    formats.write_embeddings(p, np.zeros((4, 64), np.float32))
    raw = bytearray(open(p, "rb").read())
    bad = str(tmp_path / "bad.rcbemb")
    open(bad, "wb").write(b"XXXXXXXX" + bytes(raw[8:]))
    with pytest.raises(formats.FormatError, match="magic"):
        formats.read_header(bad)
    open(bad, "wb").write(bytes(raw[:-2]))
    with pytest.raises(formats.FormatError, match="bytes"):
        formats.read_header(bad)
    with pytest.raises(formats.FormatError, match="dim"):
        formats.write_embeddings(bad, np.zeros((4, 100), np.float32))


@pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")
def test_bundle_round_trip_and_extended_report(tmp_path):
    from ragsim.config import RunConfig
    from ragsim.simulator import run
    from ragsim.workload import CorpusSpec, TraceSpec, generate_corpus, generate_trace

    rng = np.random.default_rng(np.random.SeedSequence([3]))
    corpus = generate_corpus(CorpusSpec(num_docs=300, length_mean=256.0, length_sigma=0.5,
                                        zipf_s=0.97), rng)
    trace = generate_trace(corpus, TraceSpec(duration_s=60.0, arrival_rate=0.5, k=2,
                                             prompt_tokens=32, seed=3), rng)
    emb = synth.corpus_int(corpus.num_docs).astype(np.float32)
    paths = formats.write_bundle(str(tmp_path / "run"), corpus, trace, emb)
    assert sorted(os.path.basename(p) for p in paths.values()) == \
        ["corpus.csv", "embeddings.rcbemb", "trace.jsonl"]
    c2, t2, e2 = formats.read_bundle(str(tmp_path / "run"))
    assert np.array_equal(c2.sizes, corpus.sizes) and np.allclose(c2.weights, corpus.weights)
    assert t2 == trace
    assert np.array_equal(np.asarray(e2), formats._bf16_bits(emb))
    # a trace that names a document outside the corpus is rejected
    formats.write_bundle(str(tmp_path / "bad"), corpus, trace, emb)
    with open(os.path.join(str(tmp_path / "bad"), "trace.jsonl"), "a") as fp:
        fp.write(json.dumps({"id": 10**6, "arrival_ms": 1.0, "prompt_tokens": 32,
                             "docs": [corpus.num_docs + 5], "output_tokens": 1}) + "\n")
    with pytest.raises(formats.FormatError, match="outside"):
        formats.read_bundle(str(tmp_path / "bad"))
    # the run report keeps every reference key and gains the B200 block
    cfg = RunConfig(gpu_capacity_tokens=4096, host_capacity_tokens=8192, k=2)
    rep = run(cfg, trace, corpus.size_map()).to_json(cfg)
    ext = json.loads(formats.extend_report(rep, kernels={"prefix_prefill_ms": 0.65},
                                           swap={"h2d_gbs": 54.4}, gpu="NVIDIA B200"))
    base = json.loads(rep)
    assert {k: ext[k] for k in base} == base
    assert ext["b200"]["host"]["cores_usable"] >= 1
    assert ext["b200"]["swap"]["h2d_gbs"] == 54.4


@pytest.mark.gpu
def test_retrieval_from_file_matches_in_memory(tmp_path):
    from paper_2404_12457_b200 import kernels

    n = 5000
    emb = synth.corpus_int(n, seed=2).astype(np.float32)
    p = str(tmp_path / "e.rcbemb")
    formats.write_embeddings(p, emb)
    dev = formats.load_embeddings_device(p, chunk_rows=1024)
    ref = torch.from_numpy(emb).cuda().to(torch.bfloat16)
    assert torch.equal(dev.view(torch.int16), ref.view(torch.int16))
    q = torch.randint(-100, 100, (8, synth.EMB_DIM), device="cuda").to(torch.bfloat16)
    a, _ = kernels.retrieval_topk(dev, q, 2, 4)
    b, _ = kernels.retrieval_topk(ref, q, 2, 4)
    assert torch.equal(a, b)
    # a shard: rows [1000, 3000) with global ids
    shard = formats.load_embeddings_device(p, rows=slice(1000, 3000))
    assert torch.equal(shard.view(torch.int16), ref[1000:3000].view(torch.int16))
