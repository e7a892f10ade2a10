"""GPU parity of the three hot-path kernels against the CPU oracle.

* block gather/scatter: bit-exact bytes (HBM->HBM and mapped pinned host)
* retrieval: bit-exact ids AND scores vs oracle/topk_oracle.py (integer
  embeddings make fp32 accumulation exact), ties included
* prefix-prefill attention: fp32 oracle (oracle/attn_oracle.py), tolerance
  ATTN_ATOL on bf16 outputs
* RoPE + paged KV write: fp32 oracle within bf16 rounding
"""

import math

import numpy as np
import pytest
import torch

from oracle import attn_oracle, topk_oracle
from paper_2404_12457_b200 import _lib, kernels, synth

pytestmark = pytest.mark.gpu

# bf16 output, P rounded to bf16 before PV: observed max |err| ~1e-2 on unit-scale V
ATTN_ATOL = 3e-2


def _pool(nb, L, hkv, bt, hd, seed=0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.randn((nb, L, 2, hkv, bt, hd), generator=g, device="cuda").to(torch.bfloat16)


# ---------------------------------------------------------------- block copy
# device -> device runs the TMA bulk-copy kernel: a block that is not a whole number of its
# 32 KB chunks (3 chunks + 48 B), and more units per CTA than ring stages (ring wrap)
@pytest.mark.parametrize("block_bytes,n_pairs", [(32768, 37), (2 * 1024 * 1024, 9), (4096 + 16, 300),
                                                 (3 * 32768 + 48, 11), (32768, 2000)])
def test_block_copy_hbm(block_bytes, n_pairs):
    nb = n_pairs * 2 + 3
    src = torch.randint(0, 256, (nb * block_bytes,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros_like(src)
    rng = np.random.default_rng(block_bytes)
    s = rng.permutation(nb)[:n_pairs]
    d = rng.permutation(nb)[:n_pairs]
    pairs = torch.tensor(np.stack([s, d], 1), dtype=torch.int32, device="cuda")
    kernels.block_copy(src.data_ptr(), dst.data_ptr(), block_bytes, pairs)
    torch.cuda.synchronize()
    sv = src.view(nb, block_bytes).cpu()
    dv = dst.view(nb, block_bytes).cpu()
    for a, b in zip(s, d):
        assert torch.equal(sv[a], dv[b])
    untouched = sorted(set(range(nb)) - set(d.tolist()))
    assert int(dv[untouched].abs().sum()) == 0


def test_block_copy_pinned_host_roundtrip():
    block_bytes, nb = 65536, 16
    dev = torch.randint(0, 256, (nb * block_bytes,), dtype=torch.uint8, device="cuda")
    host = torch.zeros(nb * block_bytes, dtype=torch.uint8).pin_memory()
    pairs = torch.tensor([[i, nb - 1 - i] for i in range(nb)], dtype=torch.int32, device="cuda")
    kernels.block_copy(dev.data_ptr(), host.data_ptr(), block_bytes, pairs)  # zero-copy D2H
    torch.cuda.synchronize()
    dv = dev.view(nb, block_bytes).cpu()
    hv = host.view(nb, block_bytes)
    for i in range(nb):
        assert torch.equal(dv[i], hv[nb - 1 - i])
    back = torch.zeros_like(dev)
    kernels.block_copy(host.data_ptr(), back.data_ptr(), block_bytes, pairs.flip(1))  # H2D
    torch.cuda.synchronize()
    assert torch.equal(back.cpu(), dev.cpu())


# ---------------------------------------------------------------- retrieval
@pytest.mark.parametrize("n_rows,b,k,stages", [
    (10000, 5, 2, 4), (10007, 16, 5, 4), (3000, 40, 8, 1), (20011, 64, 5, 4), (700, 64, 2, 8),
    # quad-balanced ranges / merge edge cases: empty stage segments (rows < stages), fewer rows than k,
    # ~one 32-row quad per CTA, many tiles per CTA with ragged quads
    (5, 3, 2, 8), (33, 3, 4, 8), (4741, 7, 3, 3), (150001, 64, 2, 4), (262144, 33, 1, 5),
    # > 64 queries: 2- and 4-CTA clusters sharing multicast corpus stages (ragged last CTA,
    # fewer rows than one quad per cluster, full 256)
    (20011, 65, 5, 4), (100003, 128, 2, 4), (3000, 130, 8, 1), (7, 200, 2, 3),
    (150001, 256, 2, 4),
])
def test_retrieval_scores_and_topk_exact(n_rows, b, k, stages):
    corpus = synth.corpus_int(n_rows, seed=n_rows)
    rng = np.random.default_rng(b)
    q = rng.integers(-200, 201, size=(b, synth.EMB_DIM)).astype(np.float64)
    c_dev = torch.from_numpy(corpus.astype(np.float32)).to("cuda", torch.bfloat16)
    q_dev = torch.from_numpy(q.astype(np.float32)).to("cuda", torch.bfloat16)
    scores = kernels.retrieval_scores(c_dev, q_dev).cpu().numpy()
    exact = topk_oracle.exact_scores(corpus, q)
    assert np.array_equal(scores.T.astype(np.float64), exact)
    ids, sc = kernels.retrieval_topk(c_dev, q_dev, k, stages, id_offset=1000)
    o_ids, o_sc = topk_oracle.staged_topk(corpus, q, k, stages, id_offset=1000)
    assert np.array_equal(ids.cpu().numpy(), o_ids)
    assert np.array_equal(sc.cpu().numpy().astype(np.float64), o_sc)


def test_retrieval_workspace_reuse():
    """Back-to-back calls on one workspace (different queries, scan and merge kernels
    chained by programmatic dependent launch) stay exact."""
    corpus = synth.corpus_int(30011, seed=4)
    c_dev = torch.from_numpy(corpus.astype(np.float32)).to("cuda", torch.bfloat16)
    ws = kernels.RetrievalWorkspace(corpus.shape[0], 24, 4, 4)
    outs = []
    for rep in range(5):
        q = np.random.default_rng(100 + rep).integers(-200, 201, size=(24, synth.EMB_DIM))
        q = q.astype(np.float64)
        q_dev = torch.from_numpy(q.astype(np.float32)).to("cuda", torch.bfloat16)
        outs.append((q, kernels.retrieval_topk(c_dev, q_dev, 4, 4, workspace=ws)))
    torch.cuda.synchronize()
    for q, (ids, sc) in outs:
        o_ids, o_sc = topk_oracle.staged_topk(corpus, q, 4, 4)
        assert np.array_equal(ids.cpu().numpy(), o_ids)
        assert np.array_equal(sc.cpu().numpy().astype(np.float64), o_sc)


@pytest.mark.parametrize("b", [20, 150])
def test_retrieval_ties_break_by_id(b):
    # heavy ties: rows drawn from a tiny alphabet, many duplicates (150 queries: a 4-CTA
    # cluster, ties must still break by id across the multicast CTAs' partial lists)
    rng = np.random.default_rng(3)
    base = rng.integers(-1, 2, size=(7, synth.EMB_DIM)).astype(np.int8)
    corpus = base[rng.integers(0, 7, size=5000)]
    q = rng.integers(-3, 4, size=(b, synth.EMB_DIM)).astype(np.float64)
    c_dev = torch.from_numpy(corpus.astype(np.float32)).to("cuda", torch.bfloat16)
    q_dev = torch.from_numpy(q.astype(np.float32)).to("cuda", torch.bfloat16)
    ids, sc = kernels.retrieval_topk(c_dev, q_dev, 8, 4)
    o_ids, o_sc = topk_oracle.staged_topk(corpus, q, 8, 4)
    assert np.array_equal(ids.cpu().numpy(), o_ids)


def test_retrieval_reproduces_ground_truth_docs():
    n_rows, k = 50000, 5
    corpus = synth.corpus_int(n_rows, seed=11)
    rng = np.random.default_rng(5)
    seqs = [tuple(int(x) for x in rng.choice(n_rows, size=k, replace=False)) for _ in range(48)]
    q = synth.build_queries_int(lambda ids: corpus[ids], seqs)
    c_dev = torch.from_numpy(corpus.astype(np.float32)).to("cuda", torch.bfloat16)
    q_dev = torch.from_numpy(q.astype(np.float32)).to("cuda", torch.bfloat16)
    ids, _ = kernels.retrieval_topk(c_dev, q_dev, k, 4)
    got = [tuple(int(x) for x in row) for row in ids[:, -1].cpu().numpy()]
    assert got == seqs


def test_topk_merge_shards_matches_oracle():
    rng = np.random.default_rng(9)
    shards = [synth.corpus_int(4000 + 13 * i, seed=i) for i in range(4)]
    offsets = list(np.cumsum([0] + [s.shape[0] for s in shards[:-1]]))
    q = rng.integers(-100, 101, size=(12, synth.EMB_DIM)).astype(np.float64)
    q_dev = torch.from_numpy(q.astype(np.float32)).to("cuda", torch.bfloat16)
    parts_i, parts_s = [], []
    for c, off in zip(shards, offsets):
        c_dev = torch.from_numpy(c.astype(np.float32)).to("cuda", torch.bfloat16)
        i, s = kernels.retrieval_topk(c_dev, q_dev, 5, 4, id_offset=int(off))
        parts_i.append(i)
        parts_s.append(s)
    ids, sc = kernels.topk_merge_shards(torch.stack(parts_i), torch.stack(parts_s))
    o_ids, o_sc = topk_oracle.sharded_staged_topk(shards, [int(o) for o in offsets], q, 5, 4)
    assert np.array_equal(ids.cpu().numpy(), o_ids)
    assert np.array_equal(sc.cpu().numpy().astype(np.float64), o_sc)


# ---------------------------------------------------------------- attention
def _table(segments, bt, free):
    blocks, valid = [], []
    for n in segments:
        nb = -(-n // bt)
        for i in range(nb):
            blocks.append(int(free.pop()))
            valid.append(bt if i + 1 < nb else n - (nb - 1) * bt)
    return blocks, valid


ATTN_CASES = [
    # hd, hq, hkv, bt, layers, [(prefix node sizes, suffix segment sizes)]
    (64, 4, 4, 16, 2, [([37, 100], [50, 32]), ([], [200, 32]), ([16, 16], [1])]),
    (128, 32, 8, 16, 2, [([512, 512], [32]), ([], [512, 32]), ([300], [212, 32])]),
    (128, 32, 32, 64, 1, [([512], [512, 32]), ([200, 100], [5])]),
    (128, 8, 1, 32, 1, [([77], [130, 17])]),
    (64, 8, 4, 128, 1, [([129, 3], [260])]),
    # decode steps (one new token per request over its cached context): split items
    (128, 32, 8, 64, 1, [([512, 512], [1]), ([300], [1]), ([512, 512, 512, 512], [1])]),
    # split-KV (split-only plans with few items): one request's decode step, a cached-prefix
    # prompt whose causal diagonal crosses a KV tile (fully masked rows in the last part),
    # MHA, head_dim 64 with 16-token blocks
    (128, 32, 8, 64, 1, [([4096], [1])]),
    (128, 32, 8, 64, 1, [([1020], [32])]),
    (128, 32, 32, 64, 1, [([2048], [1]), ([500], [3])]),
    (64, 8, 4, 16, 2, [([300, 200], [2])]),
    # MQA decode over a long context: 94 KV tiles -> 47 split-KV parts (> 32) in one group
    (128, 8, 1, 64, 1, [([12000], [1])]),
]


@pytest.mark.parametrize("split_kv", [False, True])
@pytest.mark.parametrize("hd,hq,hkv,bt,L,reqs", ATTN_CASES)
def test_prefix_prefill_matches_oracle(hd, hq, hkv, bt, L, reqs, split_kv):
    nb = 400
    pool = _pool(nb, L, hkv, bt, hd, seed=hd + hq + bt)
    free = list(np.random.default_rng(bt).permutation(nb))
    requests = []
    for prefix, suffix in reqs:
        blocks, valid = _table(prefix + suffix, bt, free)
        alpha, beta = sum(prefix), sum(suffix)
        requests.append((beta, alpha, blocks, valid))
    total_q = sum(r[0] for r in requests)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    q = torch.randn((total_q, hq, hd), generator=g, device="cuda").to(torch.bfloat16)
    out = torch.zeros_like(q)
    plan = kernels.AttnPlan(requests, block_tokens=bt, n_q_heads=hq, n_kv_heads=hkv,
                            split_kv=split_kv)
    for layer in range(L):
        kernels.prefix_prefill(q, out, plan, pool.data_ptr(), nb, block_tokens=bt, n_layers=L,
                               n_kv_heads=hkv, head_dim=hd, layer=layer)
        torch.cuda.synchronize()
        ref = attn_oracle.prefix_prefill(q.cpu().float(), pool.cpu(), requests, layer)
        err = (out.cpu().float() - ref).abs().max().item()
        assert err <= ATTN_ATOL, f"layer {layer}: max |err| {err}"


def test_rope_table_must_cover_the_positions():
    pool = torch.zeros((4, 1, 2, 1, 16, 64), dtype=torch.bfloat16, device="cuda")
    kv = torch.zeros((3, 64), dtype=torch.bfloat16, device="cuda")
    pos = torch.tensor([0, 1, 40], dtype=torch.int32, device="cuda")
    slots = torch.tensor([0, 1, 2], dtype=torch.int32, device="cuda")
    table = kernels.rope_table(32, 64, 1e4)
    kw = dict(block_tokens=16, n_layers=1, n_kv_heads=1, head_dim=64, layer=0, rope_theta=1e4,
              n_q_heads=1, rope=table)
    with pytest.raises(ValueError):
        kernels.kv_write_rope(None, kv, kv, None, pos, slots, pool.data_ptr(), max_pos=41, **kw)
    with pytest.raises(ValueError):
        kernels.kv_write_rope(None, kv, kv, None, pos, slots, pool.data_ptr(), **kw)


def test_split_kv_plan_splits_small_split_only_launches():
    bt = 64
    free = list(range(200))
    blocks, valid = _table([4096, 1], bt, free)
    plan = kernels.AttnPlan([(1, 4096, blocks, valid)], block_tokens=bt, n_q_heads=32,
                            n_kv_heads=8, split_kv=True)
    assert plan.work_flags == _lib.RCB_WORK_SPLIT_ONLY
    assert plan.n_combine == 8 and plan.n_work > 8 and plan.n_part_slots == plan.n_work


# ---------------------------------------------------------------- rope + kv write
def test_kv_write_rope_matches_oracle():
    hd, hq, hkv, bt, L, nb = 128, 32, 8, 16, 3, 64
    T = 70
    pool = torch.zeros((nb, L, 2, hkv, bt, hd), dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    qkv = torch.randn((T, (hq + 2 * hkv) * hd), generator=g, device="cuda").to(torch.bfloat16)
    q = qkv[:, : hq * hd]
    k = qkv[:, hq * hd:(hq + hkv) * hd]
    v = qkv[:, (hq + hkv) * hd:]
    pos = torch.arange(1000, 1000 + T, dtype=torch.int32, device="cuda")
    blocks = np.random.default_rng(0).permutation(nb)[: -(-T // bt)]
    slots = torch.tensor([int(blocks[t // bt]) * bt + t % bt for t in range(T)], dtype=torch.int32,
                         device="cuda")
    q_out = torch.empty((T, hq, hd), dtype=torch.bfloat16, device="cuda")
    kernels.kv_write_rope(q, k, v, q_out, pos, slots, pool.data_ptr(), block_tokens=bt,
                          n_layers=L, n_kv_heads=hkv, head_dim=hd, layer=1, rope_theta=10000.0)
    torch.cuda.synchronize()
    qc = q.cpu().float().view(T, hq, hd)
    kc = k.cpu().float().view(T, hkv, hd)
    q_ref = attn_oracle.apply_rope(qc, pos.cpu(), 10000.0)
    k_ref = attn_oracle.apply_rope(kc, pos.cpu(), 10000.0)
    assert (q_out.cpu().float() - q_ref).abs().max().item() < 0.05
    pc = pool.cpu()
    for t in range(T):
        b, o = int(blocks[t // bt]), t % bt
        assert (pc[b, 1, 0, :, o, :].float() - k_ref[t]).abs().max().item() < 0.05
        assert torch.equal(pc[b, 1, 1, :, o, :], v.cpu().view(T, hkv, hd)[t])
    assert int((pc[:, 0] != 0).sum()) == 0 and int((pc[:, 2] != 0).sum()) == 0


# ---------------------------------------------------------------- fused Q-RoPE
@pytest.mark.parametrize("hd,hq,hkv,bt", [(128, 32, 8, 64), (64, 4, 4, 16), (128, 8, 8, 32)])
def test_prefix_prefill_fused_rope_matches_oracle(hd, hq, hkv, bt):
    """Q read raw from a strided QKV buffer and rotated in shared memory inside the
    kernel == attention on oracle-rotated Q; K/V-only write mode leaves q untouched."""
    L, nb, theta = 1, 200, 10000.0
    pool = _pool(nb, L, hkv, bt, hd, seed=11)
    free = list(np.random.default_rng(4).permutation(nb))
    reqs = [([300, 41], [200, 32]), ([], [96]), ([512], [17])]
    requests = []
    for prefix, suffix in reqs:
        blocks, valid = _table(prefix + suffix, bt, free)
        requests.append((sum(suffix), sum(prefix), blocks, valid))
    T = sum(r[0] for r in requests)
    width = (hq + 2 * hkv) * hd
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    qkv = torch.randn((T, width), generator=g, device="cuda").to(torch.bfloat16)
    pos = torch.cat([r[1] + torch.arange(r[0]) for r in requests]).to(torch.int32)
    table = kernels.rope_table(4096, hd, theta)
    out = torch.empty((T, hq, hd), dtype=torch.bfloat16, device="cuda")
    plan = kernels.AttnPlan(requests, block_tokens=bt, n_q_heads=hq, n_kv_heads=hkv)
    kernels.prefix_prefill(qkv[:, : hq * hd], out, plan, pool.data_ptr(), nb, block_tokens=bt,
                           n_layers=L, n_kv_heads=hkv, head_dim=hd, layer=0, rope=table,
                           n_q_heads=hq)
    torch.cuda.synchronize()
    q_rot = attn_oracle.apply_rope(qkv[:, : hq * hd].cpu().float().view(T, hq, hd), pos, theta)
    ref = attn_oracle.prefix_prefill(q_rot, pool.cpu(), requests, 0)
    err = (out.cpu().float() - ref).abs().max().item()
    assert err <= ATTN_ATOL, err
    # K/V-only write: q is not rotated or written, K/V land in the pool rotated
    assert T <= nb * bt
    slots = torch.arange(T, dtype=torch.int32, device="cuda")  # token t -> block t//bt, row t%bt
    pool2 = torch.zeros_like(pool)
    kernels.kv_write_rope(None, qkv[:, hq * hd:(hq + hkv) * hd], qkv[:, (hq + hkv) * hd:], None,
                          pos.cuda(), slots, pool2.data_ptr(), block_tokens=bt, n_layers=L,
                          n_kv_heads=hkv, head_dim=hd, layer=0, rope_theta=theta, n_q_heads=hq)
    torch.cuda.synchronize()
    k_ref = attn_oracle.apply_rope(qkv[:, hq * hd:(hq + hkv) * hd].cpu().float().view(T, hkv, hd),
                                   pos, theta)
    pc = pool2.cpu()
    for t in (0, T // 2, T - 1):
        assert (pc[t // bt, 0, 0, :, t % bt, :].float() - k_ref[t]).abs().max().item() < 0.05


@pytest.mark.gpu
@pytest.mark.parametrize("with_q", [True, False])
@pytest.mark.parametrize("hq,hkv", [(32, 8), (32, 32), (40, 40)])
def test_kv_write_rope_table_is_bit_identical(with_q, hq, hkv):
    """rcb_kv_write_rope_table (cos/sin from rcb_rope_table; 8, 2 or 1 tokens per CTA as the
    row width grows: Mistral-7B, LLaMA2-7B, LLaMA2-13B K/V rows, 203 tokens so the last CTA
    is ragged) writes the same bytes as the per-token sincosf kernel: both use
    theta^(-2i/d) via exp2f + sincosf."""
    hd, bt, L, nb, T, theta = 128, 64, 2, 96, 203, 1e6
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    qkv = torch.randn((T, (hq + 2 * hkv) * hd), generator=g, device="cuda").to(torch.bfloat16)
    q = qkv[:, : hq * hd] if with_q else None
    k = qkv[:, hq * hd:(hq + hkv) * hd]
    v = qkv[:, (hq + hkv) * hd:]
    pos = (torch.randperm(5000, device="cuda")[:T] + 17).to(torch.int32)
    slots = torch.randperm(nb * bt, device="cuda")[:T].to(torch.int32)
    table = kernels.rope_table(int(pos.max()) + 1, hd, theta)
    outs = []
    for rope in (None, table):
        pool = torch.zeros((nb, L, 2, hkv, bt, hd), dtype=torch.bfloat16, device="cuda")
        q_out = torch.zeros((T, hq, hd), dtype=torch.bfloat16, device="cuda") if with_q else None
        kernels.kv_write_rope(q, k, v, q_out, pos, slots, pool.data_ptr(), block_tokens=bt,
                              n_layers=L, n_kv_heads=hkv, head_dim=hd, layer=1, rope_theta=theta,
                              n_q_heads=hq, rope=rope, max_pos=int(pos.max()) + 1)
        torch.cuda.synchronize()
        outs.append((pool, q_out))
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    if with_q:
        assert torch.equal(outs[0][1].view(torch.int16), outs[1][1].view(torch.int16))
    assert int((outs[1][0][:, 0] != 0).sum()) == 0  # layer 0 untouched


@pytest.mark.gpu
@pytest.mark.parametrize("fused_rope", [False, True])
def test_prefix_prefill_bench_shape_sampled(fused_rope):
    """The bench's step shape (Mistral-7B heads, 64-token blocks, 64 requests: 26 misses of
    1056 tokens, 26 half hits 512+544, 12 full hits 1024+32 -> pair, split and half items,
    42K query tokens) in ONE launch; one request of each kind checked against the fp32
    oracle (the whole step is too slow for the CPU oracle)."""
    hq, hkv, hd, bt, L, theta = 32, 8, 128, 64, 1, 1e6
    reqs = [(0, 1056)] * 26 + [(512, 544)] * 26 + [(1024, 32)] * 12
    n_slots = sum(-(-(a + b) // bt) for a, b in reqs)
    nb = n_slots + 16
    pool = _pool(nb, L, hkv, bt, hd, seed=21)
    free = list(np.random.default_rng(5).permutation(nb))
    requests = []
    for a, b in reqs:
        blocks, valid = _table([a + b], bt, free)
        requests.append((b, a, blocks, valid))
    T = sum(b for _, b in reqs)
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    qkv = torch.randn((T, (hq + 2 * hkv) * hd), generator=g, device="cuda").to(torch.bfloat16)
    q = qkv[:, : hq * hd]
    out = torch.empty((T, hq, hd), dtype=torch.bfloat16, device="cuda")
    plan = kernels.AttnPlan(requests, block_tokens=bt, n_q_heads=hq, n_kv_heads=hkv)
    assert (plan.tiles_q1 == 0).any() and plan.half_q0.any() and (plan.tiles_q1 > 0).any()
    rope = kernels.rope_table(plan.max_pos + 1, hd, theta) if fused_rope else None
    kernels.prefix_prefill(q, out, plan, pool.data_ptr(), nb, block_tokens=bt, n_layers=L,
                           n_kv_heads=hkv, head_dim=hd, layer=0, rope=rope, n_q_heads=hq)
    torch.cuda.synchronize()
    pool_cpu = pool.cpu()
    starts = np.cumsum([0] + [b for _, b in reqs])
    for r in (0, 30, 60):  # a miss, a half hit, a full hit
        b, a, blocks, valid = requests[r]
        qs = q[starts[r]:starts[r] + b].cpu().float().view(b, hq, hd)
        if fused_rope:
            qs = attn_oracle.apply_rope(qs, a + torch.arange(b), theta)
        ref = attn_oracle.prefix_prefill(qs, pool_cpu, [requests[r]], 0)
        got = out[starts[r]:starts[r] + b].cpu().float()
        err = (got - ref).abs().max().item()
        assert err <= ATTN_ATOL, f"request {r} (alpha {a}, beta {b}): max |err| {err}"


# ---------------------------------------------------------------- peer exchange protocol
@pytest.mark.gpu
def test_peer_window_epochs_and_bounded_wait():
    """rcb_peer_* in one process (both 'ranks' map the same window): a wait for an epoch a
    rank has not published gives up after its timeout and flags it (no device hang); once
    every rank pushed, the wait passes and the merge sees both ranks' lists in the epoch's
    parity slot."""
    import ctypes

    from paper_2404_12457_b200 import _lib

    lib = _lib.load()
    R, nq, S, k = 2, 3, 2, 2
    E = nq * S * k
    win = ctypes.c_void_p()
    assert lib.rcb_peer_window_alloc(R, E, ctypes.byref(win)) == 0
    try:
        wins = (ctypes.c_void_p * R)(win.value, win.value)
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        ids = [torch.arange(E, device="cuda").view(nq, S, k) * 10 + r for r in range(R)]
        scs = [torch.full((nq, S, k), float(r), device="cuda") for r in range(R)]
        assert lib.rcb_peer_push(wins, R, 0, E, ids[0].data_ptr(), scs[0].data_ptr(), 1, None) == 0
        out_i = torch.empty((nq, S, k), dtype=torch.int64, device="cuda")
        out_s = torch.empty((nq, S, k), dtype=torch.float32, device="cuda")
        assert lib.rcb_peer_wait(win.value, R, E, 1, 2_000_000, flag.data_ptr(), None) == 0
        torch.cuda.synchronize()
        assert int(flag.item()) == 1  # rank 1 never published epoch 1: bounded, flagged
        flag.zero_()
        assert lib.rcb_peer_push(wins, R, 1, E, ids[1].data_ptr(), scs[1].data_ptr(), 1, None) == 0
        assert lib.rcb_peer_merge(win.value, R, nq, S, k, 1, 2_000_000_000, flag.data_ptr(),
                                  out_i.data_ptr(), out_s.data_ptr(), None) == 0
        torch.cuda.synchronize()
        assert int(flag.item()) == 0
        # rank 1's scores (1.0) beat rank 0's (0.0): every merged entry comes from rank 1
        assert torch.all(out_s == 1.0) and torch.all(out_i % 10 == 1)
    finally:
        lib.rcb_peer_window_free(win)
