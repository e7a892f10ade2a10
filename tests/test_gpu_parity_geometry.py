"""Parity at the geometries the bench runs ("pin parity at the configs you bench").

(b) Cached-prefix prefill logits at Mistral-7B (GQA-4), LLaMA2-7B (MHA) and Mixtral-8x7B
    (GQA-4, 8-expert top-2 MoE FFN) geometry: head
    dim 128, 64-token blocks, full hidden size / FFN / vocab, 2 layers, 512-token documents
    (plus a ragged 300-token one for node tails), against the fp32 full-recompute oracle:
    max |logit error| <= 1e-2 (north star).
(c) One whole bench step of configs[1]: the 64 admissions the bench's planner makes
    (HotPath on the reference tree, real block tables with shared cached documents), ONE
    fused-RoPE attention launch, every request checked against the fp32 oracle.
(d) The fp32 attention oracle itself cross-checked against an independent implementation
    (flashinfer's paged prefill with LLaMA RoPE applied on the fly): pins the oracle's
    paging, RoPE convention and causal positions (q at alpha + i attends keys 0..alpha + i).

The fp32 oracles run on the GPU here (plain PyTorch fp32, TF32 off): the same arithmetic
as the host restatement, at sizes the host cannot finish in seconds.
"""

import dataclasses

import numpy as np
import pytest
import torch

from oracle import attn_oracle, model_oracle
from paper_2404_12457_b200 import kernels
from paper_2404_12457_b200.model import DIMS, PrefillModel, init_weights, suffix_slots

pytestmark = pytest.mark.gpu

LOGIT_ATOL = 1e-2
ATTN_ATOL = 3e-2


@pytest.fixture(autouse=True)
def _no_tf32():
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32 = old


@pytest.mark.parametrize("model", ["mistral-7b", "llama2-7b", "mixtral-8x7b"])
def test_cached_prefix_logits_at_bench_geometry(model):
    full = DIMS[model]
    shape = dataclasses.replace(full.shape, name=model + "-2l", n_layers=2)
    dims = dataclasses.replace(full, shape=shape)
    bt, nb = 64, 160
    w = init_weights(dims, seed=1)
    pool = torch.zeros((nb, shape.n_layers, 2, shape.n_kv_heads, bt, shape.head_dim),
                       dtype=torch.bfloat16, device="cuda")
    model_ = PrefillModel(dims, w, block_tokens=bt, num_pool_blocks=nb, pool_base=pool.data_ptr())
    g = torch.Generator().manual_seed(11)
    doc = {d: torch.randint(0, dims.vocab, (n,), generator=g)
           for d, n in ((1, 512), (2, 512), (3, 300), (4, 512))}
    free = list(np.random.default_rng(3).permutation(nb))
    node_pages = {}

    def alloc(n):
        k = -(-n // bt)
        return [int(free.pop()) for _ in range(k)], [bt] * (k - 1) + [n - (k - 1) * bt]

    def run(cached, miss, prompt):
        blocks, valid = [], []
        for d in cached:
            blocks += node_pages[d][0]
            valid += node_pages[d][1]
        alpha = sum(len(doc[d]) for d in cached)
        n_pre = len(blocks)
        segs = []
        for d in miss:
            b, v = alloc(len(doc[d]))
            segs.append((d, b, v))
            blocks += b
            valid += v
        pb, pv = alloc(len(prompt))
        blocks += pb
        valid += pv
        suffix = torch.cat([doc[d] for d in miss] + [prompt])
        beta = suffix.shape[0]
        slots, pos = suffix_slots(blocks, valid, n_pre, bt, alpha)
        plan = kernels.AttnPlan([(beta, alpha, blocks, valid)], block_tokens=bt,
                                n_q_heads=shape.n_q_heads, n_kv_heads=shape.n_kv_heads)
        logits = model_.prefill(suffix.cuda(), torch.tensor(pos, dtype=torch.int32, device="cuda"),
                                torch.tensor(slots, dtype=torch.int32, device="cuda"), plan,
                                torch.tensor([beta - 1], device="cuda"))
        for d, b, v in segs:
            node_pages[d] = (b, v)
        seq = torch.cat([doc[d] for d in cached] + [suffix])
        ref = model_oracle.forward_full(w, dims, seq, device="cuda", last_only=True)[0]
        return (logits[0] - ref).abs().max().item(), ref.abs().max().item()

    prompts = [torch.randint(0, dims.vocab, (32,), generator=g) for _ in range(4)]
    res = [run([], [1, 3], prompts[0]),   # full miss, ragged second doc (node tail)
           run([1, 3], [], prompts[1]),   # full hit over a tail block
           run([1], [2], prompts[2]),     # partial hit
           run([1, 2], [4], prompts[3])]  # two cached docs + a miss
    errs = [e for e, _ in res]
    mag = max(m for _, m in res)
    assert mag > 0.1, mag
    assert max(errs) <= LOGIT_ATOL, f"{model}: max |logit err| per request {errs} (max |logit| {mag:.3f})"


@pytest.mark.parametrize("workload,R", [("mistral7b-100k", 64), ("llama2-13b-10m", 32)])
def test_whole_bench_step_attention_against_fp32(workload, R):
    """A bench step (configs[1]: GQA-4, staged O stores; configs[3]: MHA with 40 heads, direct
    O stores and the 16-column drain): the planner's admissions after the bench's cache
    warm-up, one fused-RoPE launch, every request against the fp32 oracle."""
    from paper_2404_12457_b200.hotpath import HotPath  # puts ragsim on the path
    from paper_2404_12457_b200.pool import accounting_pool
    from paper_2404_12457_b200.workloads import WORKLOADS, make_stream, pool_blocks
    from ragsim.cost_model import synthetic_profile

    w = WORKLOADS[workload]
    n_warm = 40
    trace, sizes = make_stream(w, (n_warm + 1) * R)
    ng = pool_blocks(w.gpu_capacity_tokens, w.block_tokens, sizes.values(), R * (w.k + 1))
    hp = HotPath(w.model, gpu_capacity_tokens=w.gpu_capacity_tokens, host_capacity_tokens=0,
                 block_tokens=w.block_tokens, num_gpu_blocks=ng, num_host_blocks=0, sizes=sizes,
                 profile=synthetic_profile(), pool=accounting_pool(ng, 0, w.block_tokens))
    carry = []
    for i in range(n_warm + 1):
        batch = carry + trace[i * R:(i + 1) * R]
        adm = hp.admit_batch([(r.id, r.doc_sequence, r.prompt_tokens) for r in batch[:R]])
        carry = batch[len(adm):]
        if i < n_warm:
            for a in adm:
                hp.commit(a)
    assert len(adm) == R and any(a.alpha == 0 for a in adm)
    assert any(a.alpha > 0 for a in adm) or workload != "mistral7b-100k"
    # one layer of the step's pages, block ids remapped onto a compact pool
    s = w.model
    used = sorted({b for a in adm for b in a.blocks})
    remap = {b: i for i, b in enumerate(used)}
    requests = [(a.beta, a.alpha, [remap[b] for b in a.blocks], list(a.valid)) for a in adm]
    nb = len(used)
    g = torch.Generator(device="cuda").manual_seed(5)
    pool = torch.randn((nb, 1, 2, s.n_kv_heads, w.block_tokens, s.head_dim), generator=g,
                       device="cuda").to(torch.bfloat16)
    T = sum(r[0] for r in requests)
    qkv = torch.randn((T, s.qkv_width), generator=g, device="cuda").to(torch.bfloat16)
    plan = kernels.AttnPlan(requests, block_tokens=w.block_tokens, n_q_heads=s.n_q_heads,
                            n_kv_heads=s.n_kv_heads)
    rope = kernels.rope_table(plan.max_pos + 1, s.head_dim, s.rope_theta)
    out = torch.empty((T, s.n_q_heads, s.head_dim), dtype=torch.bfloat16, device="cuda")
    kernels.prefix_prefill(qkv[:, : s.n_q_heads * s.head_dim], out, plan, pool.data_ptr(), nb,
                           block_tokens=w.block_tokens, n_layers=1, n_kv_heads=s.n_kv_heads,
                           head_dim=s.head_dim, layer=0, rope=rope, n_q_heads=s.n_q_heads)
    torch.cuda.synchronize()
    pos = torch.cat([a + torch.arange(b) for b, a, _, _ in requests]).cuda()
    q_rot = attn_oracle.apply_rope(qkv[:, : s.n_q_heads * s.head_dim].float()
                                   .view(T, s.n_q_heads, s.head_dim), pos, s.rope_theta)
    worst = 0.0
    q0 = 0
    for r in requests:  # per request (bounded memory), all 64 of them
        ref = attn_oracle.prefix_prefill(q_rot[q0:q0 + r[0]], pool, [r], 0)
        worst = max(worst, (out[q0:q0 + r[0]].float() - ref).abs().max().item())
        q0 += r[0]
    assert worst <= ATTN_ATOL, worst


@pytest.mark.parametrize("hq,hkv", [(32, 8), (32, 32)])
def test_attention_oracle_matches_flashinfer(hq, hkv):
    """oracle (node-aligned pages with tails, RoPE by logical position, causal on logical
    positions) == flashinfer BatchPrefillWithPagedKVCacheWrapper (contiguous 16-token pages,
    pos_encoding_mode ROPE_LLAMA, causal) on the same logical K/V sequences."""
    flashinfer = pytest.importorskip("flashinfer")
    hd, theta, bt = 128, 10000.0, 64
    g = torch.Generator(device="cuda").manual_seed(2)
    shapes = [([512, 300], [544]), ([], [1056]), ([512, 512], [32]), ([77], [130, 17])]
    seqs = []
    for prefix, suffix in shapes:
        n = sum(prefix) + sum(suffix)
        k = torch.randn((n, hkv, hd), generator=g, device="cuda").to(torch.bfloat16)
        v = torch.randn((n, hkv, hd), generator=g, device="cuda").to(torch.bfloat16)
        q = torch.randn((sum(suffix), hq, hd), generator=g, device="cuda").to(torch.bfloat16)
        seqs.append((prefix, suffix, q, k, v))
    # oracle: K rotated by position into node-aligned pages (tails), Q rotated at alpha + i
    nb = sum(-(-x // bt) for p, s_, *_ in seqs for x in p + s_) + 4
    pool = torch.zeros((nb, 1, 2, hkv, bt, hd), dtype=torch.bfloat16, device="cuda")
    free = list(range(nb))
    requests, qs = [], []
    for prefix, suffix, q, k, v in seqs:
        n = k.shape[0]
        krot = attn_oracle.apply_rope(k.float(), torch.arange(n), theta).to(torch.bfloat16)
        blocks, valid, t = [], [], 0
        for seg in prefix + suffix:
            for j in range(-(-seg // bt)):
                b = free.pop(0)
                m = min(bt, seg - j * bt)
                pool[b, 0, 0, :, :m] = krot[t:t + m].transpose(0, 1)
                pool[b, 0, 1, :, :m] = v[t:t + m].transpose(0, 1)
                blocks.append(b)
                valid.append(m)
                t += m
        alpha, beta = sum(prefix), sum(suffix)
        requests.append((beta, alpha, blocks, valid))
        qs.append(attn_oracle.apply_rope(q.float(), alpha + torch.arange(beta), theta))
    ref = attn_oracle.prefix_prefill(torch.cat(qs), pool, requests, 0)
    # flashinfer: unrotated K/V in contiguous 16-token pages, RoPE applied inside
    ps = 16
    pages, indptr, last, qo = [], [0], [], [0]
    for _, _, q, k, v in seqs:
        n = k.shape[0]
        npg = -(-n // ps)
        kp = torch.zeros((npg * ps, hkv, hd), dtype=torch.bfloat16, device="cuda")
        vp = torch.zeros_like(kp)
        kp[:n], vp[:n] = k, v
        pages.append(torch.stack([kp.view(npg, ps, hkv, hd), vp.view(npg, ps, hkv, hd)], dim=1))
        indptr.append(indptr[-1] + npg)
        last.append(n - (npg - 1) * ps)
        qo.append(qo[-1] + q.shape[0])
    kv_cache = torch.cat(pages)
    i32 = lambda x: torch.tensor(x, dtype=torch.int32, device="cuda")  # noqa: E731
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    try:
        wrap = flashinfer.BatchPrefillWithPagedKVCacheWrapper(ws, "NHD")
        wrap.plan(i32(qo), i32(indptr), torch.arange(indptr[-1], dtype=torch.int32, device="cuda"),
                  i32(last), hq, hkv, hd, ps, causal=True, pos_encoding_mode="ROPE_LLAMA",
                  rope_theta=theta, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        fi = wrap.run(torch.cat([s[2] for s in seqs]), kv_cache)
    except Exception as exc:  # JIT toolchain problems on the box are not oracle failures
        pytest.skip(f"flashinfer paged prefill unavailable: {type(exc).__name__}: {exc}"[:300])
    err = (fi.float() - ref).abs().max().item()
    assert err <= ATTN_ATOL, err
