"""Layer-pipelined swap-in: per-layer-group DMAs + per-layer fences.

The reference charges a host-tier hit serially, ``transfer_ms + prefill_ms``
(simulator.py:505-510).  ``BlockPool.flush_layered`` issues the pending swap-in
batch one layer group at a time and ``fence_layer(l)`` makes a layer's attention
wait only for its own group, so the copy of the later layers overlaps the
earlier layers' compute.  These tests check that the bytes are exactly those of
the whole-block path, that each fence orders the reads of its layer, and that a
cached-prefix prefill fed this way gives the same logits as the serial path.
"""

import numpy as np
import pytest
import torch

from oracle import model_oracle
from paper_2404_12457_b200 import _lib, kernels
from paper_2404_12457_b200.model import DIMS, PrefillModel, init_weights, suffix_slots
from paper_2404_12457_b200.pool import BlockPool

pytestmark = pytest.mark.gpu

LOGIT_ATOL = 1e-2


def _geom(n_layers):
    return dict(block_tokens=16, n_layers=n_layers, n_kv_heads=2, head_dim=64)


@pytest.mark.parametrize("n_layers,lpg", [(6, 4), (6, 1), (5, 5), (3, 8)])
def test_layered_swap_in_bytes_and_fences(n_layers, lpg):
    geom = _geom(n_layers)
    bb = n_layers * 2 * 2 * 16 * 64 * 2
    nb = 48
    u8 = torch.zeros((nb, bb), dtype=torch.uint8, device="cuda")
    pool = BlockPool(nb, 32, gpu_base=u8.data_ptr(), swap_mode=_lib.RCB_SWAP_DMA, **geom)
    # fragment the free list so swap-in runs are non-contiguous (several DMA runs)
    pool.node_alloc_gpu(1, 70)   # 5 blocks
    pool.node_alloc_gpu(2, 16)   # 1 block
    pool.node_alloc_gpu(3, 40)   # 3 blocks
    u8.copy_(torch.randint(0, 256, u8.shape, dtype=torch.uint8, device="cuda"))
    want = {k: u8[pool.node_blocks(k)].clone() for k in (1, 3)}
    pool.node_swap_out([1, 3])
    pool.sync()
    pool.node_alloc_gpu(4, 20)   # takes the lowest freed blocks: 1 and 3 land elsewhere
    u8.zero_()
    torch.cuda.synchronize()
    pool.node_swap_in([1, 3])
    stream = torch.cuda.current_stream()
    pool.flush_layered(lpg)
    lb = bb // n_layers
    got = {k: torch.empty_like(want[k]) for k in want}
    for layer in range(n_layers):
        pool.fence_layer(layer, stream)  # reads of this layer ordered after its group only
        for k in want:
            blocks = pool.node_blocks(k)
            got[k][:, layer * lb:(layer + 1) * lb] = u8[blocks, layer * lb:(layer + 1) * lb]
    torch.cuda.synchronize()
    for k in want:
        assert torch.equal(got[k], want[k]), f"node {k}: layered swap-in bytes differ"
    st = pool.stats()
    assert st["h2d_bytes"] == (5 + 3) * bb
    pool.close()


@pytest.mark.parametrize("lpg", [1, 2, 6])
def test_layered_swap_out_with_block_reuse(lpg):
    """Swap-outs off the critical path: a swap-out and a swap-in pending in ONE batch,
    issued per layer group (swap-outs first in every group).  A new node reuses the
    swapped-out node's blocks and writes them layer by layer, each layer fenced on its
    group only: the host copy still holds the old bytes, the swap-in lands intact, and
    the new writes survive."""
    n_layers = 6
    geom = _geom(n_layers)
    bb = n_layers * 2 * 2 * 16 * 64 * 2
    lb = bb // n_layers
    nb = 32
    u8 = torch.zeros((nb, bb), dtype=torch.uint8, device="cuda")
    pool = BlockPool(nb, 32, gpu_base=u8.data_ptr(), swap_mode=_lib.RCB_SWAP_STAGED, **geom)
    pool.node_alloc_gpu(1, 70)   # blocks 0-4
    pool.node_alloc_gpu(2, 16)   # block 5
    pool.node_alloc_gpu(3, 40)   # blocks 6-8
    u8.copy_(torch.randint(0, 256, u8.shape, dtype=torch.uint8, device="cuda"))
    want1 = u8[pool.node_blocks(1)].clone()
    want3 = u8[pool.node_blocks(3)].clone()
    pool.node_swap_out([3])
    pool.sync()
    # one batch: swap-out 1, a new node 4 takes 1's freed blocks, swap-in 3
    pool.node_swap_out([1])
    pool.node_alloc_gpu(4, 70)
    assert pool.node_blocks(4) == [0, 1, 2, 3, 4]
    pool.node_swap_in([3])
    stream = torch.cuda.current_stream()
    pool.flush_layered(lpg)
    new4 = torch.randint(0, 256, (5, bb), dtype=torch.uint8, device="cuda")
    b4 = pool.node_blocks(4)
    for layer in range(n_layers):
        pool.fence_layer(layer, stream)  # the K/V write of this layer into reused blocks
        u8[b4, layer * lb:(layer + 1) * lb] = new4[:, layer * lb:(layer + 1) * lb]
    torch.cuda.synchronize()
    st = pool.stats()
    assert st["d2h_bytes"] == (3 + 5) * bb and st["h2d_bytes"] == 3 * bb
    assert torch.equal(u8[pool.node_blocks(3)], want3), "swap-in bytes differ"
    assert torch.equal(u8[b4], new4), "reused blocks lost the new writes"
    pool.wait_for(stream)
    pool.node_free_gpu(2)
    pool.node_swap_in([1])  # the host copy written by the layered swap-out
    pool.sync()
    assert torch.equal(u8[pool.node_blocks(1)], want1), "layered swap-out bytes differ"
    pool.close()


def test_layered_flush_of_swap_outs_and_plain_fence():
    geom = _geom(4)
    pool = BlockPool(16, 8, swap_mode=_lib.RCB_SWAP_STAGED, **geom)
    pool.node_alloc_gpu(1, 30)
    pool.node_swap_out([1])
    pool.flush_layered(2)  # pending D2H: two layer groups
    pool.fence_layer(3, torch.cuda.current_stream())
    pool.flush()
    pool.fence_layer(3, torch.cuda.current_stream())  # no layered batch outstanding: full fence
    pool.drain()
    assert pool.stats()["d2h_bytes"] == 2 * pool.block_bytes
    with pytest.raises(Exception):
        pool.fence_layer(4, torch.cuda.current_stream())
    pool.close()


def test_layered_prefill_matches_serial_and_full_recompute():
    """Docs computed by request A are swapped out, then swapped back in for request B
    with a layered flush; B's logits equal the serial-fence run bit for bit and the
    fp32 full recomputation within LOGIT_ATOL."""
    dims = DIMS["tiny"]
    s = dims.shape
    bt, nb = 16, 128
    w = init_weights(dims, seed=0)
    kv = torch.zeros((nb, s.n_layers, 2, s.n_kv_heads, bt, s.head_dim), dtype=torch.bfloat16,
                     device="cuda")
    pool = BlockPool(nb, 64, block_tokens=bt, n_layers=s.n_layers, n_kv_heads=s.n_kv_heads,
                     head_dim=s.head_dim, gpu_base=kv.data_ptr(), swap_mode=_lib.RCB_SWAP_DMA)
    model = PrefillModel(dims, w, block_tokens=bt, num_pool_blocks=nb, pool_base=kv.data_ptr())
    g = torch.Generator().manual_seed(5)
    docs = {1: torch.randint(0, dims.vocab, (45,), generator=g),
            2: torch.randint(0, dims.vocab, (83,), generator=g)}
    prompts = [torch.randint(0, dims.vocab, (32,), generator=g) for _ in range(3)]
    stream = torch.cuda.current_stream()

    def table(keys):
        blocks, valid = pool.block_table(keys)
        return blocks, valid

    def prefill(cached, miss, prompt, prompt_key, fence=None):
        blocks, valid = table(cached + miss + [prompt_key])
        alpha = sum(len(docs[d]) for d in cached)
        n_pre = sum(-(-len(docs[d]) // bt) for d in cached)
        suffix = torch.cat([docs[d] for d in miss] + [prompt])
        beta = suffix.shape[0]
        slots, pos = suffix_slots(blocks, valid, n_pre, bt, alpha)
        plan = kernels.AttnPlan([(beta, alpha, blocks, valid)], block_tokens=bt,
                                n_q_heads=s.n_q_heads, n_kv_heads=s.n_kv_heads)
        return model.prefill(suffix.cuda(), torch.tensor(pos, dtype=torch.int32, device="cuda"),
                             torch.tensor(slots, dtype=torch.int32, device="cuda"), plan,
                             torch.tensor([beta - 1], device="cuda"), layer_fence=fence)[0]

    # A: computes both docs into node pages 1, 2 (+ prompt node 10)
    for k in (1, 2):
        pool.node_alloc_gpu(k, len(docs[k]))
    pool.node_alloc_gpu(10, 32)
    prefill([], [1, 2], prompts[0], 10)
    pool.wait_for(stream)
    pool.node_swap_out([1, 2])
    pool.sync()
    kv.zero_()  # the cached pages must come back from the host tier
    torch.cuda.synchronize()

    # B, layered: swap in, one group per layer, attention of layer l fenced on group l
    pool.node_alloc_gpu(11, 32)
    pool.node_swap_in([1, 2])
    pool.flush_layered(1)
    logits_layered = prefill([1, 2], [], prompts[1], 11,
                             fence=lambda layer: pool.fence_layer(layer, stream))
    # B again, serial: pages already resident, full fence
    pool.node_alloc_gpu(12, 32)
    pool.fence_into(stream)
    logits_serial = prefill([1, 2], [], prompts[1], 12)
    torch.cuda.synchronize()
    assert torch.equal(logits_layered, logits_serial)
    ref = model_oracle.forward_full(w, dims, torch.cat([docs[1], docs[2], prompts[1]]))[-1]
    err = (logits_layered.cpu() - ref).abs().max().item()
    assert err <= LOGIT_ATOL, f"max |logit err| {err}"
    pool.close()
