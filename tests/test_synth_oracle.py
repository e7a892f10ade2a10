"""CPU checks of the real synthetic corpus and the margin-aware top-k oracle
(the checker behind tests/test_retrieval_real.py and smoke())."""

import numpy as np
import torch

from oracle import topk_oracle
from paper_2404_12457_b200 import synth


def test_host_and_device_generators_agree_bitwise():
    a = synth.corpus_f32(3000, seed=9, row_offset=12345)
    b = synth.corpus_device(3000, seed=9, row_offset=12345, device="cpu", chunk=700)
    assert np.array_equal(a, b.float().numpy())


def test_real_rows_are_unit_norm_gaussian_like_bf16():
    a = synth.corpus_f32(4000, seed=1)
    assert np.array_equal(a, synth.to_bf16_f32(a))  # bf16 values
    norms = np.linalg.norm(a.astype(np.float64), axis=1)
    assert np.abs(norms - 1).max() < 2e-3
    z = a.reshape(-1) * np.sqrt(synth.EMB_DIM)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    assert 2.65 < (z ** 4).mean() < 2.75  # Irwin-Hall(4): kurtosis 3 - 6/20 = 2.7 (normal: 3)


def test_queries_reproduce_targets_with_margin():
    n = 20000
    corpus = synth.corpus_f32(n, seed=2)
    rng = np.random.default_rng(4)
    for k in (2, 5):
        docs = [tuple(int(x) for x in rng.choice(n, size=k, replace=False)) for _ in range(20)]
        q = synth.build_queries(lambda ids: corpus[ids], docs, seed=k)
        assert np.array_equal(q, synth.to_bf16_f32(q))
        s64 = topk_oracle.exact_scores(corpus, q)
        bound = topk_oracle.acc_bound(q)
        for qi, d in enumerate(docs):
            r_ids, r_sc = topk_oracle.stage_ranking(s64[qi], np.arange(n), k)
            assert tuple(r_ids[:k]) == d
            assert (r_sc[:-1] - r_sc[1:]).min() > 50 * bound[qi]  # final stage never ambiguous


def test_fp32_accumulation_stays_within_the_bound():
    """Sequential fp32 sums (forward, reverse, pairwise-by-64) of bf16 products differ
    from float64 by less than acc_bound: the bound the GPU tests rely on."""
    corpus = synth.corpus_f32(2000, seed=3)
    rng = np.random.default_rng(0)
    q = synth.build_queries(lambda ids: corpus[ids],
                            [tuple(rng.choice(2000, size=2, replace=False)) for _ in range(8)])
    bound = topk_oracle.acc_bound(q)
    s64 = topk_oracle.exact_scores(corpus, q)
    prods = (q[:, None, :].astype(np.float32) * corpus[None, :, :])  # exact in fp32
    fwd = np.zeros(prods.shape[:2], dtype=np.float32)
    for i in range(prods.shape[2]):
        fwd = fwd + prods[:, :, i]
    rev = np.zeros_like(fwd)
    for i in reversed(range(prods.shape[2])):
        rev = rev + prods[:, :, i]
    blk = prods.reshape(*prods.shape[:2], -1, 64).sum(axis=3, dtype=np.float32).sum(
        axis=2, dtype=np.float32)
    for approx in (fwd, rev, blk):
        err = np.abs(approx.astype(np.float64) - s64).max(axis=1)
        assert (err <= bound / 4).all(), (err, bound)


def test_margin_oracle_flags_ambiguous_stages_and_tolerates_them():
    rng = np.random.default_rng(1)
    scores = rng.standard_normal((3, 400)) * 0.05
    scores[0, 10] = scores[0, 20] = 0.9  # exact tie at the top: ambiguous order
    scores[1, 5] = 0.9
    scores[1, 6] = 0.9 - 1e-9  # below 2 * bound: ambiguous
    scores[2, 7] = 0.9
    scores[2, 8] = 0.5  # clear
    bound = np.full(3, 1e-6)
    ids, sc, amb, kth = topk_oracle.staged_topk_margin(scores, 2, 1, bound)
    assert amb[0, 0] and amb[1, 0]
    assert list(ids[0, 0]) == [10, 20]  # id asc on ties
    s2 = scores[2].copy()
    s2[[7, 8]] = -1
    third = np.sort(s2)[-1]
    assert amb[2, 0] == bool(0.5 - third <= 2e-6)
    # a swapped order within the bound is accepted; a non-member is not
    ok = topk_oracle.check_topk_tolerant([6, 5], [0.9, 0.9], lambda i: scores[1, i], kth[1, 0], 1e-6)
    assert ok == []
    bad = topk_oracle.check_topk_tolerant([5, 3], [0.9, float(scores[1, 3])],
                                          lambda i: scores[1, i], kth[1, 0], 1e-6)
    assert any("below the k-th" in e for e in bad)
    dup = topk_oracle.check_topk_tolerant([5, 5], [0.9, 0.9], lambda i: scores[1, i], kth[1, 0], 1e-6)
    assert any("duplicate" in e for e in dup)


def test_staged_from_scores_matches_staged_topk_on_integer_corpus():
    corpus = synth.corpus_int(3001, seed=4)
    q = np.random.default_rng(2).integers(-50, 51, size=(6, synth.EMB_DIM)).astype(np.float64)
    a = topk_oracle.staged_topk(corpus, q, 3, 4, id_offset=7)
    b = topk_oracle.staged_topk_from_scores(topk_oracle.exact_scores(corpus, q), 3, 4, id_offset=7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
