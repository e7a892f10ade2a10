"""BlockPool — Python handle on the native paged doc-KV pool (rcb_pool_*).

Event interface (shared with oracle/block_oracle.BlockOracle so the two can
be driven by the same knowledge-tree event stream and compared):

    node_alloc_gpu(key, tokens)      node_free_gpu(key)      node_free_host(key)
    node_swap_out(keys)              node_swap_in(keys)
    gen_reserve(gen, seg_tokens)     gen_free_segment(gen, seg)
    node_adopt(key, gen, seg)        gen_release(gen)
    node_blocks(key, tier) -> list   block_table(node_keys, gen) -> (blocks, valid)

Keys are KnowledgeNode.serial (ragsim tree.py:94-96).  Status 1 (out of
blocks) raises PoolCapacityError, which the tree layer maps onto ragsim's
InsufficientEvictableCapacity (tree.py:49-50); anything else is PoolError.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import (RCB_ERR_NO_BLOCKS, RCB_OK, RCB_POOL_ACCOUNTING, RCB_SWAP_STAGED,
                   RCB_TIER_GPU, RCB_TIER_HOST, load)

GPU = RCB_TIER_GPU
HOST = RCB_TIER_HOST


class PoolError(RuntimeError):
    pass


class PoolCapacityError(PoolError):
    pass


def blocks_for(tokens: int, block_tokens: int) -> int:
    return -(-int(tokens) // block_tokens)


class BlockPool:
    def __init__(self, num_gpu_blocks: int, num_host_blocks: int, *, block_tokens: int,
                 n_layers: int, n_kv_heads: int, head_dim: int, elem_bytes: int = 2,
                 swap_mode: int = RCB_SWAP_STAGED, gpu_base: int | None = None,
                 copy_stream=None) -> None:
        self._lib = load()
        self.block_tokens = block_tokens
        self.n_layers = n_layers
        self.n_kv_heads = n_kv_heads
        self.head_dim = head_dim
        self.elem_bytes = elem_bytes
        self.num_gpu_blocks = num_gpu_blocks
        self.num_host_blocks = num_host_blocks
        self.swap_mode = swap_mode
        self.block_bytes = n_layers * 2 * n_kv_heads * block_tokens * head_dim * elem_bytes
        handle = ctypes.c_void_p()
        self._check(self._lib.rcb_pool_create(
            num_gpu_blocks, num_host_blocks, block_tokens, n_layers, n_kv_heads, head_dim,
            elem_bytes, swap_mode, gpu_base or None, _lib.stream_handle(copy_stream) or None,
            ctypes.byref(handle)), "rcb_pool_create")
        self._h = handle
        self._buf = (ctypes.c_int32 * 1)()
        self._cap = 0

    # ------------------------------------------------------------------ plumbing
    def _check(self, code: int, what: str) -> None:
        if code == RCB_OK:
            return
        msg = self._lib.rcb_last_error().decode(errors="replace")
        if code == RCB_ERR_NO_BLOCKS:
            raise PoolCapacityError(f"{what}: {msg}")
        raise PoolError(f"{what} (status {code}): {msg}")

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.rcb_pool_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:
            pass

    def _out(self, n: int):
        if n > self._cap:
            self._cap = max(n, 2 * self._cap, 1024)
            self._buf = (ctypes.c_int32 * self._cap)()
            self._buf2 = (ctypes.c_int32 * self._cap)()
        return self._buf

    def info(self) -> dict:
        out = (ctypes.c_int64 * 7)()
        self._check(self._lib.rcb_pool_info(self._h, out), "rcb_pool_info")
        return {"gpu_base": out[0], "host_base": out[1], "block_bytes": out[2],
                "gpu_free": out[3], "host_free": out[4], "num_gpu": out[5], "num_host": out[6]}

    def stats(self) -> dict:
        out = (ctypes.c_int64 * 8)()
        self._check(self._lib.rcb_pool_stats(self._h, out), "rcb_pool_stats")
        keys = ("swap_out_blocks", "swap_in_blocks", "d2h_bytes", "h2d_bytes", "swap_out_calls",
                "swap_in_calls", "kernel_launches", "memcpy_calls")
        return dict(zip(keys, list(out)))

    @property
    def gpu_base(self) -> int:
        return self.info()["gpu_base"]

    @property
    def host_base(self) -> int:
        return self.info()["host_base"]

    def host_view(self) -> np.ndarray:
        """numpy uint8 [num_host_blocks, block_bytes] view of the pinned host tier."""
        base = self.host_base
        n = self.num_host_blocks * self.block_bytes
        arr = (ctypes.c_uint8 * n).from_address(base)
        return np.ctypeslib.as_array(arr).reshape(self.num_host_blocks, self.block_bytes)

    def set_swap_mode(self, mode: int) -> None:
        self._check(self._lib.rcb_pool_set_swap_mode(self._h, mode), "rcb_pool_set_swap_mode")
        self.swap_mode = mode

    # ------------------------------------------------------------------ events
    def node_alloc_gpu(self, key: int, tokens: int) -> None:
        self._check(self._lib.rcb_node_alloc_gpu(self._h, key, tokens), "node_alloc_gpu")

    def node_free_gpu(self, key: int) -> None:
        self._check(self._lib.rcb_node_free_gpu(self._h, key), "node_free_gpu")

    def node_free_host(self, key: int) -> None:
        self._check(self._lib.rcb_node_free_host(self._h, key), "node_free_host")

    def node_swap_out(self, keys) -> None:
        arr = _lib.i64_array(keys)
        self._check(self._lib.rcb_node_swap_out(self._h, arr, len(keys)), "node_swap_out")

    def node_swap_in(self, keys) -> None:
        arr = _lib.i64_array(keys)
        self._check(self._lib.rcb_node_swap_in(self._h, arr, len(keys)), "node_swap_in")

    def gen_reserve(self, gen: int, seg_tokens) -> None:
        arr = _lib.i32_array(seg_tokens)
        self._check(self._lib.rcb_gen_reserve(self._h, gen, arr, len(seg_tokens)), "gen_reserve")

    def gen_free_segment(self, gen: int, seg: int) -> None:
        self._check(self._lib.rcb_gen_free_segment(self._h, gen, seg), "gen_free_segment")

    def node_adopt(self, key: int, gen: int, seg: int) -> None:
        self._check(self._lib.rcb_node_adopt(self._h, key, gen, seg), "node_adopt")

    def gen_release(self, gen: int) -> None:
        self._check(self._lib.rcb_gen_release(self._h, gen), "gen_release")

    # ------------------------------------------------------------------ queries
    def node_blocks(self, key: int, tier: int = GPU) -> list[int]:
        n = ctypes.c_int32()
        buf = self._out(4096)
        code = self._lib.rcb_node_blocks(self._h, key, tier, buf, self._cap, ctypes.byref(n))
        if code != RCB_OK and n.value > self._cap:
            buf = self._out(n.value)
            code = self._lib.rcb_node_blocks(self._h, key, tier, buf, self._cap, ctypes.byref(n))
        self._check(code, "node_blocks")
        return list(buf[: n.value])

    def gen_blocks(self, gen: int, seg: int) -> list[int]:
        n = ctypes.c_int32()
        buf = self._out(4096)
        code = self._lib.rcb_gen_blocks(self._h, gen, seg, buf, self._cap, ctypes.byref(n))
        if code != RCB_OK and n.value > self._cap:
            buf = self._out(n.value)
            code = self._lib.rcb_gen_blocks(self._h, gen, seg, buf, self._cap, ctypes.byref(n))
        self._check(code, "gen_blocks")
        return list(buf[: n.value])

    def block_table(self, node_keys, gen: int = -1) -> tuple[list[int], list[int]]:
        keys = _lib.i64_array(node_keys)
        n = ctypes.c_int32()
        cap = max(4096, self._cap)
        self._out(cap)
        code = self._lib.rcb_block_table(self._h, keys, len(node_keys), gen, self._buf,
                                         self._buf2, self._cap, ctypes.byref(n))
        if code != RCB_OK and n.value == 0 and self._cap < self.num_gpu_blocks:
            self._out(self.num_gpu_blocks)
            code = self._lib.rcb_block_table(self._h, keys, len(node_keys), gen, self._buf,
                                             self._buf2, self._cap, ctypes.byref(n))
        self._check(code, "block_table")
        return list(self._buf[: n.value]), list(self._buf2[: n.value])

    # ------------------------------------------------------------------ ordering
    def flush(self) -> None:
        self._check(self._lib.rcb_pool_flush(self._h), "rcb_pool_flush")

    def fence_into(self, stream) -> None:
        self._check(self._lib.rcb_pool_fence_into(self._h, _lib.stream_handle(stream)),
                    "rcb_pool_fence_into")

    def wait_for(self, stream) -> None:
        self._check(self._lib.rcb_pool_wait_for(self._h, _lib.stream_handle(stream)),
                    "rcb_pool_wait_for")

    def flush_layered(self, layers_per_group: int) -> None:
        """Issue a pending swap-in batch as per-layer-group DMAs."""
        self._check(self._lib.rcb_pool_flush_layered(self._h, layers_per_group),
                    "rcb_pool_flush_layered")

    def fence_layer(self, layer: int, stream) -> None:
        self._check(self._lib.rcb_pool_fence_layer(self._h, layer, _lib.stream_handle(stream)),
                    "rcb_pool_fence_layer")

    def drain(self) -> None:
        self._check(self._lib.rcb_pool_drain(self._h), "rcb_pool_drain")

    def sync(self) -> None:
        self._check(self._lib.rcb_pool_sync(self._h), "rcb_pool_sync")


def accounting_pool(num_gpu_blocks: int, num_host_blocks: int, block_tokens: int) -> BlockPool:
    """Native allocator with no device memory (decision/block-table work on CPU)."""
    return BlockPool(num_gpu_blocks, num_host_blocks, block_tokens=block_tokens, n_layers=1,
                     n_kv_heads=1, head_dim=8, swap_mode=RCB_POOL_ACCOUNTING)
