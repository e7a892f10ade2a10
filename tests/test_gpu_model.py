"""Cached-prefix prefill reproduces full recomputation (logits, tiny model).

Request A computes docs d1, d2 and a prompt from scratch, writing their KV
into node-aligned pool pages (with tails).  Requests B and C then reuse the
cached pages (B: both docs cached; C: d1 cached, d3 missing) and compute
only their suffix.  Every request's last-token logits must match the fp32
full-sequence oracle within LOGIT_ATOL (north star: <= 1e-2).
"""

import numpy as np
import pytest
import torch

from oracle import model_oracle
from paper_2404_12457_b200 import kernels
from paper_2404_12457_b200.model import DIMS, PrefillModel, init_weights, suffix_slots

pytestmark = pytest.mark.gpu

LOGIT_ATOL = 1e-2


def test_cached_prefix_prefill_matches_full_recompute():
    dims = DIMS["tiny"]
    s = dims.shape
    bt, nb = 16, 256
    w = init_weights(dims, seed=0)
    pool = torch.zeros((nb, s.n_layers, 2, s.n_kv_heads, bt, s.head_dim), dtype=torch.bfloat16,
                       device="cuda")
    model = PrefillModel(dims, w, block_tokens=bt, num_pool_blocks=nb, pool_base=pool.data_ptr())
    g = torch.Generator().manual_seed(3)
    doc = {d: torch.randint(0, dims.vocab, (n,), generator=g) for d, n in ((1, 37), (2, 100), (3, 60))}
    prompts = [torch.randint(0, dims.vocab, (32,), generator=g) for _ in range(3)]
    free = list(np.random.default_rng(0).permutation(nb))

    def alloc(n):
        k = -(-n // bt)
        blocks = [int(free.pop()) for _ in range(k)]
        return blocks, [bt] * (k - 1) + [n - (k - 1) * bt]

    node_pages = {}

    def run(cached_docs, miss_docs, prompt):
        blocks, valid = [], []
        for d in cached_docs:
            blocks += node_pages[d][0]
            valid += node_pages[d][1]
        alpha = sum(len(doc[d]) for d in cached_docs)
        n_pre = len(blocks)
        segs = []
        for d in miss_docs:
            b, v = alloc(len(doc[d]))
            segs.append((d, b, v))
            blocks += b
            valid += v
        pb, pv = alloc(len(prompt))
        blocks += pb
        valid += pv
        suffix = torch.cat([doc[d] for d in miss_docs] + [prompt])
        beta = suffix.shape[0]
        slots, pos = suffix_slots(blocks, valid, n_pre, bt, alpha)
        plan = kernels.AttnPlan([(beta, alpha, blocks, valid)], block_tokens=bt,
                                n_q_heads=s.n_q_heads, n_kv_heads=s.n_kv_heads)
        logits = model.prefill(suffix.cuda(), torch.tensor(pos, dtype=torch.int32, device="cuda"),
                               torch.tensor(slots, dtype=torch.int32, device="cuda"), plan,
                               torch.tensor([beta - 1], device="cuda"))
        for d, b, v in segs:
            node_pages[d] = (b, v)  # the committed node adopts its pages
        full = torch.cat([doc[d] for d in cached_docs] + [suffix])
        ref = model_oracle.forward_full(w, dims, full)[-1]
        return (logits[0].cpu() - ref).abs().max().item(), ref.abs().max().item()

    err_a, mag = run([], [1, 2], prompts[0])
    err_b, _ = run([1, 2], [], prompts[1])
    err_c, _ = run([1], [3], prompts[2])
    assert mag > 0.1  # logits are not trivially small
    errs = (err_a, err_b, err_c)
    assert max(errs) <= LOGIT_ATOL, f"max |logit err| per request {errs} (max |logit| {mag:.3f})"


@pytest.mark.parametrize("t,d", [(1, 4096), (37, 256), (300, 5120)])
def test_fused_rmsnorm_residual_and_silu_mul(t, d):
    """rcb_rmsnorm_residual / rcb_silu_mul vs the fp32 torch expressions they replace
    (model.py before the fusion): residual exact in fp32, outputs within one bf16 ulp."""
    g = torch.Generator(device="cpu").manual_seed(t)
    x = torch.randn((t, d), generator=g).cuda()
    add = torch.randn((t, d), generator=g).cuda().to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(d, generator=g)).cuda().to(torch.bfloat16)
    x_ref = x + add.float()
    h_ref = (x_ref * torch.rsqrt(x_ref.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float())
    h = kernels.rmsnorm_residual(x, add, w, 1e-5)
    torch.cuda.synchronize()
    assert torch.equal(x, x_ref)
    assert (h.float() - h_ref).abs().max().item() <= 1e-2 * h_ref.abs().max().item()
    gu = torch.randn((t, 2 * d), generator=g).cuda().to(torch.bfloat16)
    a_ref = torch.nn.functional.silu(gu[:, :d].float()) * gu[:, d:].float()
    a = kernels.silu_mul(gu)
    assert (a.float() - a_ref).abs().max().item() <= 1e-2 * a_ref.abs().max().item()
