"""Small launches of every kernel variant, for compute-sanitizer (memcheck / racecheck /
synccheck).  Each launch is checked against the oracle so a sanitizer run is also a parity
run.  Usage:  compute-sanitizer --tool racecheck python tools/sanitize_kernels.py
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import attn_oracle, topk_oracle  # noqa: E402
from paper_2404_12457_b200 import kernels, synth  # noqa: E402
from paper_2404_12457_b200.pool import BlockPool  # noqa: E402


def table(segs, bt, free):
    blocks, valid = [], []
    for n in segs:
        for j in range(-(-n // bt)):
            blocks.append(free.pop())
            valid.append(min(bt, n - j * bt))
    return blocks, valid


def attention(hq, hkv, hd, bt, shapes, rope, split_kv=False):
    nb = 64
    g = torch.Generator(device="cuda").manual_seed(hq * hkv + bt)
    pool = torch.randn((nb, 1, 2, hkv, bt, hd), generator=g, device="cuda").to(torch.bfloat16)
    free = list(range(nb))
    reqs = []
    for prefix, suffix in shapes:
        b, v = table(prefix + suffix, bt, free)
        reqs.append((sum(suffix), sum(prefix), b, v))
    T = sum(r[0] for r in reqs)
    qkv = torch.randn((T, (hq + 2 * hkv) * hd), generator=g, device="cuda").to(torch.bfloat16)
    q = qkv[:, : hq * hd]
    out = torch.empty((T, hq, hd), dtype=torch.bfloat16, device="cuda")
    plan = kernels.AttnPlan(reqs, block_tokens=bt, n_q_heads=hq, n_kv_heads=hkv, split_kv=split_kv)
    tab = kernels.rope_table(max(plan.max_pos, 2) + 1, hd, 1e4) if rope else None
    kernels.prefix_prefill(q if rope else q.contiguous().view(T, hq, hd), out, plan,
                           pool.data_ptr(), nb, block_tokens=bt, n_layers=1, n_kv_heads=hkv,
                           head_dim=hd, layer=0, rope=tab, n_q_heads=hq)
    torch.cuda.synchronize()
    qf = q.float().reshape(T, hq, hd)
    if rope:
        pos = torch.cat([a + torch.arange(b) for b, a, _, _ in reqs])
        qf = attn_oracle.apply_rope(qf.cpu(), pos, 1e4)
    ref = attn_oracle.prefix_prefill(qf.cpu(), pool.cpu(), reqs, 0)
    err = (out.cpu().float() - ref).abs().max().item()
    assert err < 3e-2, err
    return err


def main():
    torch.cuda.set_device(0)
    errs = {}
    # attention: pair items + causal half tiles (GQA, fused RoPE), MHA, split-only decode,
    # split-KV parts + combine
    errs["gqa_rope"] = attention(32, 8, 128, 64, [([200], [300, 32]), ([], [160])], rope=True)
    errs["mha"] = attention(8, 8, 128, 32, [([64], [130])], rope=False)
    # MHA with fused RoPE: direct O stores, Q(ii+2) landing right after item ii's last QK
    errs["mha_rope"] = attention(4, 4, 128, 64, [([], [544]), ([128], [300]), ([], [130])],
                                 rope=True)
    errs["decode"] = attention(32, 8, 128, 64, [([500], [1]), ([300], [1])], rope=True)
    errs["split_kv"] = attention(8, 1, 128, 64, [([1500], [1])], rope=False, split_kv=True)
    # retrieval scan + merge, shard merge
    corpus = synth.corpus_f32(5000, seed=2)
    docs = [(3, 17), (4000, 12), (99, 4999)]
    qs = synth.build_queries(lambda ids: corpus[ids], docs)
    c = torch.from_numpy(corpus).cuda().to(torch.bfloat16)
    qd = torch.from_numpy(qs).cuda().to(torch.bfloat16)
    ids, sc = kernels.retrieval_topk(c, qd, 2, 4)
    assert [tuple(r) for r in ids[:, -1].cpu().tolist()] == docs
    m_ids, _ = kernels.topk_merge_shards(torch.stack([ids, ids]), torch.stack([sc, sc]))
    assert torch.equal(m_ids[:, -1], ids[:, -1])
    # HBM -> HBM block copy (TMA bulk kernel), ragged last chunk, ring wrap
    bb, npairs = 3 * 32768 + 48, 40
    src = torch.randint(0, 256, (2 * npairs * bb,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros_like(src)
    pr = torch.stack([torch.arange(npairs), torch.arange(2 * npairs - 1, npairs - 1, -1)], 1)
    kernels.block_copy(src.data_ptr(), dst.data_ptr(), bb, pr.to(torch.int32).cuda())
    torch.cuda.synchronize()
    sv, dv = src.view(2 * npairs, bb), dst.view(2 * npairs, bb)
    assert torch.equal(sv[pr[:, 0].cuda()], dv[pr[:, 1].cuda()])
    # K/V write (table-driven) + pool swaps (staged gather/scatter kernels + DMA)
    bt, L, hkv, hd = 16, 2, 4, 64
    pool_t = torch.zeros((32, L, 2, hkv, bt, hd), dtype=torch.bfloat16, device="cuda")
    kv = torch.randn((40, 2 * hkv * hd), device="cuda").to(torch.bfloat16)
    pos = torch.arange(40, dtype=torch.int32, device="cuda")
    slots = torch.arange(40, dtype=torch.int32, device="cuda")
    kernels.kv_write_rope(None, kv[:, : hkv * hd], kv[:, hkv * hd:], None, pos, slots,
                          pool_t.data_ptr(), block_tokens=bt, n_layers=L, n_kv_heads=hkv,
                          head_dim=hd, layer=1, rope_theta=1e4, n_q_heads=hkv,
                          rope=kernels.rope_table(64, hd, 1e4), max_pos=40)
    bp = BlockPool(32, 16, gpu_base=pool_t.data_ptr(), block_tokens=bt, n_layers=L,
                   n_kv_heads=hkv, head_dim=hd)
    bp.node_alloc_gpu(1, 40)
    before = pool_t[bp.node_blocks(1, 0)].clone()
    bp.node_swap_out([1])
    bp.node_swap_in([1])
    bp.sync()
    assert torch.equal(pool_t[bp.node_blocks(1, 0)], before)
    bp.close()
    torch.cuda.synchronize()
    print("sanitize_kernels ok:", {k: round(v, 4) for k, v in errs.items()})


if __name__ == "__main__":
    main()
