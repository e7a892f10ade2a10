"""Thin torch-facing wrappers over the C-ABI kernels.

torch is used only as device-memory/stream plumbing: every call passes raw
pointers to libragcache_b200.so (include/ragcache_b200.h).  No CPU path: a
missing library raises RcbUnavailable, a non-CUDA tensor raises ValueError.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import _lib
from ._lib import check, load


def _dev_ptr(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise ValueError("rcb kernels take CUDA tensors only (no CPU fallback)")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return _lib.stream_handle(stream)


class _PinnedRing:
    """Reusable pinned staging buffers for the per-step host -> device uploads (block
    tables, work lists, slot maps).  ``Tensor.pin_memory()`` per upload goes through the
    caching host allocator, which cannot reuse a block while its copy is in flight and
    falls back to cudaHostAlloc (milliseconds, and it can serialise with the device);
    here a buffer is reused once the event recorded after its last copy has completed,
    and grows (power of two) only when an upload outgrows it."""

    def __init__(self, depth: int = 8) -> None:
        self.bufs: list[torch.Tensor | None] = [None] * depth
        self.events: list[torch.cuda.Event | None] = [None] * depth
        self.i = 0

    def upload(self, t: torch.Tensor, device) -> torch.Tensor:
        i = self.i
        self.i = (i + 1) % len(self.bufs)
        if self.events[i] is not None:
            self.events[i].synchronize()  # its previous copy has left the buffer
        n = t.numel() * t.element_size()
        buf = self.bufs[i]
        if buf is None or buf.numel() < n:
            buf = torch.empty(max(1 << 16, 1 << (n - 1).bit_length()), dtype=torch.uint8).pin_memory()
            self.bufs[i] = buf
        host = buf[:n].view(t.dtype).view(t.shape)
        host.copy_(t)
        out = host.to(device, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.events[i] = ev
        return out


_ring: _PinnedRing | None = None


def _upload(arr: np.ndarray, device) -> torch.Tensor:
    """Host array -> device without a stream sync: a pageable copy would wait for the
    work already queued (e.g. the previous step's prefill) before returning."""
    global _ring
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if torch.device(device).type != "cuda":
        return t.to(device)
    if _ring is None:
        _ring = _PinnedRing()
    return _ring.upload(t, device)


def block_copy(src_base: int, dst_base: int, block_bytes: int, pairs: torch.Tensor,
               stream=None) -> None:
    """dst[pairs[i,1]] = src[pairs[i,0]] for block_bytes-sized blocks (device/mapped ptrs)."""
    pairs = pairs.to(dtype=torch.int32).contiguous()
    check(load().rcb_kv_block_copy(src_base, dst_base, block_bytes, _dev_ptr(pairs),
                                   pairs.shape[0], _stream(stream)), "rcb_kv_block_copy")


def rope_table(max_pos: int, head_dim: int, rope_theta: float, device="cuda",
               stream=None) -> torch.Tensor:
    """float32 [max_pos, head_dim/2, 2] = (cos, sin) for fused-RoPE prefill."""
    t = torch.empty((max_pos, head_dim // 2, 2), dtype=torch.float32, device=device)
    check(load().rcb_rope_table(_dev_ptr(t), max_pos, head_dim, float(rope_theta),
                                _stream(stream)), "rcb_rope_table")
    return t


def kv_write_rope(q, k: torch.Tensor, v: torch.Tensor, q_out, positions: torch.Tensor,
                  slots: torch.Tensor, pool_base: int, *, block_tokens: int, n_layers: int,
                  n_kv_heads: int, head_dim: int, layer: int, rope_theta: float,
                  n_q_heads: int | None = None, rope: torch.Tensor | None = None,
                  max_pos: int | None = None, stream=None) -> None:
    """RoPE q,k then scatter k,v into the pool (q/k/v may be strided row views).
    q = q_out = None: K/V only (Q is rotated inside prefix_prefill).  With ``rope`` (an
    rcb_rope_table) cos/sin are read from it instead of being recomputed per token
    (identical values); ``max_pos`` (exclusive bound of ``positions``, e.g.
    AttnPlan.max_pos) is then required and must be covered by the table: the kernel
    indexes the table by position without a bounds check."""
    n_tokens = k.shape[0]
    if n_q_heads is None:
        n_q_heads = q_out.shape[1]
    assert k.stride(-1) == 1 and v.stride(-1) == 1 and k.stride(0) == v.stride(0)
    if q is not None:
        assert q.stride(-1) == 1
    if rope is not None:  # cos/sin from an rcb_rope_table (covering every position)
        if rope.dtype != torch.float32 or rope.shape[1] * 2 != head_dim:
            raise ValueError(f"rope table {tuple(rope.shape)} does not match head_dim {head_dim}")
        if max_pos is None or rope.shape[0] < max_pos:
            raise ValueError(f"rope table of {rope.shape[0]} rows must cover positions < max_pos "
                             f"({max_pos}; pass the positions' exclusive bound)")
        check(load().rcb_kv_write_rope_table(
            _dev_ptr(q) if q is not None else None, q.stride(0) if q is not None else 0,
            _dev_ptr(k), _dev_ptr(v), k.stride(0),
            _dev_ptr(q_out) if q_out is not None else None,
            _dev_ptr(positions), _dev_ptr(slots), n_tokens, n_q_heads, pool_base, block_tokens,
            n_layers, n_kv_heads, head_dim, layer, _dev_ptr(rope), _stream(stream)),
            "rcb_kv_write_rope_table")
        return
    check(load().rcb_kv_write_rope(
        _dev_ptr(q) if q is not None else None, q.stride(0) if q is not None else 0,
        _dev_ptr(k), _dev_ptr(v), k.stride(0),
        _dev_ptr(q_out) if q_out is not None else None,
        _dev_ptr(positions), _dev_ptr(slots), n_tokens, n_q_heads, pool_base, block_tokens,
        n_layers, n_kv_heads, head_dim, layer, float(rope_theta), _stream(stream)),
        "rcb_kv_write_rope")


def _num_sms(device) -> int:
    try:
        return torch.cuda.get_device_properties(torch.device(device)).multi_processor_count
    except (RuntimeError, AssertionError, ValueError):
        return 148


def _split_kv(items: np.ndarray, n_sms: int, bpt: int, tq: int):
    """Split-KV for split-only plans with few items (one request's decode step or
    cached-prefix prefill: one item per KV head would leave most SMs idle).  Opt-in:
    on B200 a single Mistral-7B request measured 27.6 us split vs 18.4 us unsplit (decode,
    1056-token context) -- the per-CTA prologue and the combine launch outweigh the
    parallelism at these sizes.  Each item's
    KV tiles are cut into P contiguous parts (>= 2 tiles, so both softmax warpgroups
    work); a part writes fp32 (O, max, sum) to its slot and one combine group per split
    item merges them (rcb_prefix_prefill combine_dev).  Returns (items, groups)."""
    target = max(1, n_sms // len(items))
    out, groups, slot = [], [], 0
    for it in items:
        packed = int(np.uint32(it[7]))
        n0, half0 = packed & 0x7FFF, (packed >> 15) & 1
        parts = max(1, min(target, n0 // 2))
        if parts == 1:
            out.append(it.copy())
            continue
        cuts = [round(k * n0 / parts) for k in range(parts + 1)]
        for k in range(parts):
            t0, t1 = cuts[k], cuts[k + 1]
            sub = it.copy()
            sub[3] = it[3] + t0 * bpt
            sub[4] = min(int(it[4]) - t0 * bpt, (t1 - t0) * bpt)
            sub[6] = int(it[6]) | ((slot + k + 1) << 8)
            sub[7] = np.uint32((t1 - t0) | ((half0 if t1 == n0 else 0) << 15)).view(np.int32)
            out.append(sub)
        # {q_start, q_len, tok_base, kv_head, slot0, n_parts}
        groups.append([it[0], it[1], 2 * it[5] * tq, it[6], slot, parts])
        slot += parts
    items = np.stack(out).astype(np.int32)
    order = np.argsort(-(items[:, 7].view(np.uint32) & 0x7FFF), kind="stable")  # heaviest first
    return items[order], np.asarray(groups, dtype=np.int32).reshape(-1, 6)


class AttnPlan:
    """Device-resident block tables + work list for one prefill batch.

    requests: list of (q_len, q_pos0, blocks, valid) — blocks/valid are the
    request's block table (cached prefix nodes then suffix segments) as
    produced by BlockPool.block_table.
    """

    def __init__(self, requests, *, block_tokens: int, n_q_heads: int, n_kv_heads: int,
                 device="cuda", split_kv: bool | None = None) -> None:
        meta = []
        ids: list[int] = []
        valid: list[int] = []
        pos: list[int] = []
        q_start = 0
        for q_len, q_pos0, blocks, vals in requests:
            meta.extend([q_start, q_len, q_pos0, len(ids), len(blocks)])
            acc = 0
            for b, v in zip(blocks, vals):
                ids.append(int(b))
                valid.append(int(v))
                pos.append(acc)
                acc += int(v)
            if acc != q_pos0 + q_len:
                raise ValueError(f"block table covers {acc} tokens, expected {q_pos0 + q_len}")
            q_start += q_len
        self.total_q = q_start
        self.n_req = len(requests)
        self.max_pos = max((r[1] + r[0] for r in requests), default=0)
        meta_np = np.asarray(meta, dtype=np.int32)
        valid_np = np.asarray(valid, dtype=np.int32)
        pos_np = np.asarray(pos, dtype=np.int32)
        g = n_q_heads // n_kv_heads
        cap = sum(max(0, -(-r[0] // (256 // g))) for r in requests) * n_kv_heads + 1
        work = np.zeros(cap * 8, dtype=np.int32)
        n_work = np.zeros(1, dtype=np.int32)
        check(load().rcb_attn_plan(
            meta_np.ctypes.data_as(_lib._p32), self.n_req, valid_np.ctypes.data_as(_lib._p32),
            pos_np.ctypes.data_as(_lib._p32), block_tokens, n_q_heads, n_kv_heads,
            work.ctypes.data_as(_lib._p32), cap, n_work.ctypes.data_as(_lib._p32)),
            "rcb_attn_plan")
        self.n_work = int(n_work[0])
        # {q_start, q_len, q_pos0, blk_begin, blk_count, q_pair, kv_head,
        #  n0 | half0 << 15 | n1 << 16 | half1 << 31}: an item = two adjacent 128-row query
        # tiles sharing each KV tile it loads; half_w: Q_w's last KV tile needs 64 slots
        self.work_host = work[: self.n_work * 8].reshape(-1, 8)
        packed = self.work_host[:, 7].view(np.uint32)
        self.tiles_q0 = (packed & 0x7FFF).astype(np.int64)
        self.tiles_q1 = ((packed >> 16) & 0x7FFF).astype(np.int64)
        self.half_q0 = ((packed >> 15) & 1).astype(bool)
        self.half_q1 = ((packed >> 31) & 1).astype(bool)
        self.kv_tiles = int(np.maximum(self.tiles_q0, self.tiles_q1).sum()) if self.n_work else 0
        # every item a lone query tile (decode, short prompts over cached docs): the kernel
        # variant with one Q tile per item buffer and a deeper K/V ring
        self.work_flags = _lib.RCB_WORK_SPLIT_ONLY if not self.tiles_q1.any() else 0
        self.mma_tiles = int((self.tiles_q0 + self.tiles_q1).sum()) if self.n_work else 0
        items = work[: self.n_work * 8].reshape(-1, 8)
        groups = np.zeros((0, 6), dtype=np.int32)
        self.n_part_slots = 0
        if split_kv is None:  # opt-in: measured slower at the sizes it targets
            split_kv = bool(os.environ.get("RCB_SPLIT_KV"))
        if split_kv and self.work_flags and 0 < self.n_work and 2 * self.n_work <= _num_sms(device):
            items, groups = _split_kv(items, _num_sms(device), 128 // block_tokens, 128 // g)
            self.n_part_slots = int(groups[:, 5].sum()) if len(groups) else 0
        self.n_work = items.shape[0]
        self.n_combine = groups.shape[0]
        # work items first: the kernel reads them as int4 (16-byte aligned)
        pack = np.concatenate([items.reshape(-1), meta_np, np.asarray(ids, dtype=np.int32),
                               valid_np, pos_np, groups.reshape(-1)])
        self._buf = _upload(pack, device)
        o = 0
        self.work = self._buf[o:o + self.n_work * 8]; o += self.n_work * 8
        self.meta = self._buf[o:o + meta_np.size]; o += meta_np.size
        self.blk_ids = self._buf[o:o + len(ids)]; o += len(ids)
        self.blk_valid = self._buf[o:o + len(ids)]; o += len(ids)
        self.blk_pos = self._buf[o:o + len(ids)]; o += len(ids)
        self.combine = self._buf[o:o + groups.size]
        self.part_ws = None  # fp32 split-KV parts, sized on first use (needs head_dim)
        self.requests = requests


def _part_ws(plan: AttnPlan, head_dim: int, device) -> torch.Tensor:
    need = plan.n_part_slots * 128 * (8 + 4 * head_dim)
    if plan.part_ws is None or plan.part_ws.numel() < need:
        plan.part_ws = torch.empty(need, dtype=torch.uint8, device=device)
    return plan.part_ws


def prefix_prefill(q: torch.Tensor, out: torch.Tensor, plan: AttnPlan, pool_base: int,
                   num_pool_blocks: int, *, block_tokens: int, n_layers: int, n_kv_heads: int,
                   head_dim: int, layer: int, softmax_scale: float | None = None,
                   rope: torch.Tensor | None = None, n_q_heads: int | None = None,
                   stream=None) -> None:
    """Prefix-aware prefill attention for one layer (tcgen05 kernel).

    q: [T, Hq, d] rotated queries, or (with ``rope``, a rope_table) the raw query
    columns of the QKV projection: a [T, >= Hq*d] row view whose RoPE is applied
    in shared memory inside the kernel."""
    assert q.dtype == torch.bfloat16 and out.is_contiguous() and q.stride(-1) == 1
    if n_q_heads is None:
        n_q_heads = out.shape[1]
    row_stride = q.stride(0)
    if rope is not None and (rope.dtype != torch.float32 or rope.shape[0] < max(plan.max_pos, 2)
                             or rope.shape[1] * 2 != head_dim):  # row 1 seeds the angle steps
        raise ValueError(f"rope table {tuple(rope.shape)} does not cover positions < "
                         f"{plan.max_pos} at head_dim {head_dim}")
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(head_dim)
    check(load().rcb_prefix_prefill(
        _dev_ptr(q), row_stride, _dev_ptr(out), q.shape[0], n_q_heads, pool_base,
        num_pool_blocks, block_tokens, n_layers, n_kv_heads, head_dim, layer,
        _dev_ptr(plan.meta), _dev_ptr(plan.blk_ids), _dev_ptr(plan.blk_valid),
        _dev_ptr(plan.blk_pos), _dev_ptr(plan.work), plan.n_work, float(softmax_scale),
        _dev_ptr(rope) if rope is not None else None, plan.work_flags,
        _dev_ptr(_part_ws(plan, head_dim, out.device)) if plan.n_part_slots else None,
        plan.n_part_slots, _dev_ptr(plan.combine) if plan.n_combine else None, plan.n_combine,
        _stream(stream)), "rcb_prefix_prefill")


def rmsnorm_residual(x: torch.Tensor, add: torch.Tensor | None, weight: torch.Tensor,
                     eps: float, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """x (fp32 [T, d], updated in place) += add (bf16); returns bf16 rmsnorm(x) * weight."""
    assert x.dtype == torch.float32 and x.is_contiguous() and weight.dtype == torch.bfloat16
    if add is not None:
        assert add.dtype == torch.bfloat16 and add.is_contiguous() and add.shape == x.shape
    if out is None:
        out = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    check(load().rcb_rmsnorm_residual(
        _dev_ptr(x), _dev_ptr(add) if add is not None else None, _dev_ptr(weight), _dev_ptr(out),
        x.shape[0], x.shape[1], float(eps), _stream(stream)), "rcb_rmsnorm_residual")
    return out


def silu_mul(gate_up: torch.Tensor, stream=None) -> torch.Tensor:
    """gate_up bf16 [T, 2F] -> bf16 silu(gate) * up [T, F]."""
    assert gate_up.dtype == torch.bfloat16 and gate_up.is_contiguous()
    t, f2 = gate_up.shape
    out = torch.empty((t, f2 // 2), dtype=torch.bfloat16, device=gate_up.device)
    check(load().rcb_silu_mul(_dev_ptr(gate_up), _dev_ptr(out), t, f2 // 2, _stream(stream)),
          "rcb_silu_mul")
    return out


MAX_SCAN_QUERIES = 256  # queries per rcb_retrieval_topk call (retrieval.cu kMaxQueries; > 64 runs as
#                         a 2- or 4-CTA cluster sharing each multicast corpus stage)


class RetrievalWorkspace:
    def __init__(self, n_rows: int, n_queries: int, k: int, n_stages: int, device="cuda"):
        self.nbytes = int(load().rcb_retrieval_workspace_bytes(n_rows, n_queries, k, n_stages))
        self.buf = torch.empty(max(16, self.nbytes), dtype=torch.uint8, device=device)
        self.key = (n_rows, n_queries, k, n_stages)


def retrieval_topk(corpus: torch.Tensor, queries: torch.Tensor, k: int, n_stages: int,
                   id_offset: int = 0, workspace: RetrievalWorkspace | None = None,
                   ids_out: torch.Tensor | None = None, scores_out: torch.Tensor | None = None,
                   stream=None):
    """Staged exact top-k: returns (ids int64 [b,S,k], scores fp32 [b,S,k])."""
    assert corpus.dtype == torch.bfloat16 and queries.dtype == torch.bfloat16
    n_rows, dim = corpus.shape
    b = queries.shape[0]
    if workspace is None or workspace.key != (n_rows, b, k, n_stages):
        workspace = RetrievalWorkspace(n_rows, b, k, n_stages, corpus.device)
    if ids_out is None:
        ids_out = torch.empty((b, n_stages, k), dtype=torch.int64, device=corpus.device)
    if scores_out is None:
        scores_out = torch.empty((b, n_stages, k), dtype=torch.float32, device=corpus.device)
    check(load().rcb_retrieval_topk(
        _dev_ptr(corpus), n_rows, dim, _dev_ptr(queries), b, k, n_stages, id_offset,
        _dev_ptr(workspace.buf), workspace.nbytes, _dev_ptr(ids_out), _dev_ptr(scores_out),
        _stream(stream)), "rcb_retrieval_topk")
    return ids_out, scores_out


def retrieval_scores(corpus: torch.Tensor, queries: torch.Tensor, stream=None) -> torch.Tensor:
    n_rows, dim = corpus.shape
    b = queries.shape[0]
    out = torch.empty((n_rows, b), dtype=torch.float32, device=corpus.device)
    check(load().rcb_retrieval_scores(_dev_ptr(corpus), n_rows, dim, _dev_ptr(queries), b,
                                      _dev_ptr(out), _stream(stream)), "rcb_retrieval_scores")
    return out


def topk_merge_shards(ids: torch.Tensor, scores: torch.Tensor, stream=None):
    """ids/scores [n_shards, b, S, k] -> merged [b, S, k] (score desc, id asc)."""
    n_shards, b, s, k = ids.shape
    ids = ids.contiguous()
    scores = scores.contiguous()
    ids_out = torch.empty((b, s, k), dtype=torch.int64, device=ids.device)
    sc_out = torch.empty((b, s, k), dtype=torch.float32, device=ids.device)
    check(load().rcb_topk_merge_shards(_dev_ptr(ids), _dev_ptr(scores), n_shards, b, s, k,
                                       _dev_ptr(ids_out), _dev_ptr(sc_out), _stream(stream)),
          "rcb_topk_merge_shards")
    return ids_out, sc_out


class _DeviceView:
    """__cuda_array_interface__ over a raw device range (a view into a peer window)."""

    def __init__(self, ptr: int, shape, typestr: str) -> None:
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class PeerExchange:
    """Exchange over peer memory (rcb_peer_*, csrc/peer.cu).

    Each rank allocates an exchange window of ``n_entries`` 8-byte slots per (parity, rank),
    exports it as a CUDA IPC handle, all-gathers the handles once
    (``comm.all_gather_object``) and maps every peer's window (NVLink P2P on one box; the
    same memory when ranks share a GPU).  Two uses:

    * ``merge(ids, scores)`` (``lists=(n_queries, S, k)``): push this rank's staged lists
      into slot (epoch & 1, rank) of every window, publish the epoch, wait for all ranks'
      epochs and merge the own window -- one push + one merge kernel instead of two
      all-gathers + the merge;
    * ``gather(x)``: a raw all-gather of x's bytes; returns a view of the own window's slot
      holding every rank's rows in rank order.

    Successive calls of one window alternate parity slots; a rank reuses a slot only two
    epochs later, after a later exchange of the same step sequence has completed on every
    rank (ShardedRetriever: queries(e+2) are pushed after lists(e+1) arrived from all ranks,
    which each rank pushes after scanning queries(e+1), i.e. after it finished with (e)).
    """

    def __init__(self, comm, n_entries: int, *, lists=None, timeout_s: float = 10.0,
                 device="cuda") -> None:
        lib = load()
        self.lib = lib
        self.R, self.rank = comm.world, comm.rank
        self.E = int(n_entries)
        if lists is not None:
            self.nq, self.S, self.k = lists
            assert self.E == self.nq * self.S * self.k
        self.timeout_ns = int(timeout_s * 1e9)
        self.own = None
        self.opened = []
        # every rank reaches both agreement rounds whatever fails locally, so the ranks
        # either all use the windows or all raise (a split decision would deadlock the next
        # collective against a peer spinning on its window)
        handle = None
        try:
            win = ctypes.c_void_p()
            check(lib.rcb_peer_window_alloc(self.R, self.E, ctypes.byref(win)),
                  "rcb_peer_window_alloc")
            self.own = win.value
            h = (ctypes.c_uint8 * _lib.RCB_PEER_HANDLE_BYTES)()
            check(lib.rcb_peer_ipc_handle(self.own, h), "rcb_peer_ipc_handle")
            handle = bytes(h)
        except RuntimeError as exc:
            err = str(exc)
        handles = comm.all_gather_object(handle)
        if any(hb is None for hb in handles):
            self.close()
            raise RuntimeError(f"peer window export failed on rank(s) "
                               f"{[r for r, hb in enumerate(handles) if hb is None]}"
                               + (f": {err}" if handle is None else ""))
        wins, ok = [], True
        for r, hb in enumerate(handles):
            if r == self.rank:
                wins.append(self.own)
                continue
            p = ctypes.c_void_p()
            buf = (ctypes.c_uint8 * len(hb)).from_buffer_copy(hb)
            if lib.rcb_peer_open(buf, ctypes.byref(p)) != 0:
                ok = False
                break
            self.opened.append(p.value)
            wins.append(p.value)
        oks = comm.all_gather_object(ok)
        if not all(oks):
            self.close()
            raise RuntimeError(f"peer window mapping failed on rank(s) "
                               f"{[r for r, o in enumerate(oks) if not o]}")
        self.windows = (ctypes.c_void_p * self.R)(*wins)
        self.epoch = 0
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=device)

    def merge(self, ids: torch.Tensor, scores: torch.Tensor, stream=None):
        """ids int64 / scores f32 [n_queries, S, k] of this rank's shard -> merged lists."""
        assert ids.shape == (self.nq, self.S, self.k) and ids.is_contiguous() and scores.is_contiguous()
        self.epoch += 1
        st = _stream(stream)
        check(self.lib.rcb_peer_push(self.windows, self.R, self.rank, self.E, _dev_ptr(ids),
                                     _dev_ptr(scores), self.epoch, st), "rcb_peer_push")
        ids_out = torch.empty_like(ids)
        sc_out = torch.empty_like(scores)
        check(self.lib.rcb_peer_merge(self.own, self.R, self.nq, self.S, self.k, self.epoch,
                                      self.timeout_ns, _dev_ptr(self.timed_out),
                                      _dev_ptr(ids_out), _dev_ptr(sc_out), st), "rcb_peer_merge")
        return ids_out, sc_out

    def gather(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        """All-gather of a contiguous device tensor (every rank the same shape, 8E bytes):
        a [world * x.shape[0], *x.shape[1:]] view of the own window (valid until the slot's
        next reuse, two calls later)."""
        nbytes = x.numel() * x.element_size()
        assert x.is_contiguous() and nbytes == 8 * self.E
        self.epoch += 1
        st = _stream(stream)
        check(self.lib.rcb_peer_push_bytes(self.windows, self.R, self.rank, self.E, _dev_ptr(x),
                                           nbytes, self.epoch, st), "rcb_peer_push_bytes")
        check(self.lib.rcb_peer_wait(self.own, self.R, self.E, self.epoch, self.timeout_ns,
                                     _dev_ptr(self.timed_out), st), "rcb_peer_wait")
        off = self.lib.rcb_peer_slot_offset(self.R, self.E, self.epoch)
        words = torch.as_tensor(_DeviceView(self.own + off, (self.R * self.E,), "<i8"),
                                device=x.device)
        return words.view(x.dtype).view((self.R * x.shape[0],) + tuple(x.shape[1:]))

    def check_timeout(self) -> None:
        """Raise if any wait gave up on a peer (reads a device flag: syncs)."""
        if int(self.timed_out.item()):
            raise RuntimeError("peer exchange: a rank's data did not arrive within the timeout")

    def close(self) -> None:
        for p in self.opened:
            self.lib.rcb_peer_close(ctypes.c_void_p(p))
        self.opened = []
        if self.own:
            self.lib.rcb_peer_window_free(ctypes.c_void_p(self.own))
            self.own = None
