"""ctypes binding of libragcache_b200.so (the C-ABI declared in include/ragcache_b200.h).

This is the reference-side binding a ragsim maintainer would add: the
reference is pure Python (ragsim, /root/reference/pkg/src/ragsim) and has no
FFI of its own, so its tier transitions, prefill and retrieval stand-ins are
bound here.  There is no fallback: if the shared library is missing the
import fails loudly (``RcbUnavailable``).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

LIB_NAME = "libragcache_b200.so"
# RCB_LIB_PATH selects an alternate in-tree build (A/B kernel experiments only)
LIB_PATH = os.environ.get("RCB_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

RCB_OK = 0
RCB_ERR_NO_BLOCKS = 1
RCB_ERR_BAD_HANDLE = 2
RCB_ERR_CUDA = 3
RCB_ERR_ARG = 4
RCB_PEER_HANDLE_BYTES = 64

RCB_TIER_GPU = 0
RCB_TIER_HOST = 1

RCB_SWAP_STAGED = 0
RCB_SWAP_ZEROCOPY = 1
RCB_SWAP_DMA = 2
RCB_POOL_ACCOUNTING = 3

RCB_WORK_SPLIT_ONLY = 1


class RcbUnavailable(RuntimeError):
    """The native library is not built / cannot be loaded (no CPU fallback exists)."""


class RcbError(RuntimeError):
    def __init__(self, code: int, msg: str) -> None:
        super().__init__(f"rcb status {code}: {msg}")
        self.code = code


_p32 = POINTER(c_int32)
_p64 = POINTER(c_int64)

# (name, restype, argtypes) — must match include/ragcache_b200.h exactly
SIGNATURES = [
    ("rcb_last_error", c_char_p, []),
    ("rcb_version", c_int, []),
    ("rcb_pool_create", c_int, [c_int64, c_int64, c_int32, c_int32, c_int32, c_int32, c_int32,
                                c_int32, c_void_p, c_void_p, POINTER(c_void_p)]),
    ("rcb_pool_destroy", c_int, [c_void_p]),
    ("rcb_pool_info", c_int, [c_void_p, _p64]),
    ("rcb_pool_stats", c_int, [c_void_p, _p64]),
    ("rcb_pool_set_swap_mode", c_int, [c_void_p, c_int32]),
    ("rcb_node_alloc_gpu", c_int, [c_void_p, c_int64, c_int32]),
    ("rcb_node_free_gpu", c_int, [c_void_p, c_int64]),
    ("rcb_node_free_host", c_int, [c_void_p, c_int64]),
    ("rcb_node_swap_out", c_int, [c_void_p, _p64, c_int32]),
    ("rcb_node_swap_in", c_int, [c_void_p, _p64, c_int32]),
    ("rcb_gen_reserve", c_int, [c_void_p, c_int64, _p32, c_int32]),
    ("rcb_node_adopt", c_int, [c_void_p, c_int64, c_int64, c_int32]),
    ("rcb_gen_free_segment", c_int, [c_void_p, c_int64, c_int32]),
    ("rcb_gen_release", c_int, [c_void_p, c_int64]),
    ("rcb_node_blocks", c_int, [c_void_p, c_int64, c_int32, _p32, c_int32, _p32]),
    ("rcb_gen_blocks", c_int, [c_void_p, c_int64, c_int32, _p32, c_int32, _p32]),
    ("rcb_block_table", c_int, [c_void_p, _p64, c_int32, c_int64, _p32, _p32, c_int32, _p32]),
    ("rcb_pool_flush", c_int, [c_void_p]),
    ("rcb_pool_fence_into", c_int, [c_void_p, c_void_p]),
    ("rcb_pool_wait_for", c_int, [c_void_p, c_void_p]),
    ("rcb_pool_sync", c_int, [c_void_p]),
    ("rcb_pool_flush_layered", c_int, [c_void_p, c_int32]),
    ("rcb_pool_fence_layer", c_int, [c_void_p, c_int32, c_void_p]),
    ("rcb_pool_drain", c_int, [c_void_p]),
    ("rcb_kv_block_copy", c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int32, c_void_p]),
    ("rcb_kv_write_rope", c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p,
                                  c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_int32,
                                  c_int32, c_int32, c_int32, c_int32, c_float, c_void_p]),
    ("rcb_kv_write_rope_table", c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                                        c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p,
                                        c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p,
                                        c_void_p]),
    ("rcb_rope_table", c_int, [c_void_p, c_int32, c_int32, c_float, c_void_p]),
    ("rcb_prefix_prefill", c_int, [c_void_p, c_int64, c_void_p, c_int32, c_int32, c_void_p,
                                   c_int64, c_int32, c_int32, c_int32, c_int32, c_int32,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                                   c_float, c_void_p, c_int32, c_void_p, c_int32, c_void_p,
                                   c_int32, c_void_p]),
    ("rcb_rmsnorm_residual", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32,
                                     c_float, c_void_p]),
    ("rcb_silu_mul", c_int, [c_void_p, c_void_p, c_int32, c_int32, c_void_p]),
    ("rcb_attn_plan", c_int, [_p32, c_int32, _p32, _p32, c_int32, c_int32, c_int32, _p32,
                              c_int32, _p32]),
    ("rcb_retrieval_workspace_bytes", c_int64, [c_int64, c_int32, c_int32, c_int32]),
    ("rcb_retrieval_topk", c_int, [c_void_p, c_int64, c_int32, c_void_p, c_int32, c_int32,
                                   c_int32, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
                                   c_void_p]),
    ("rcb_retrieval_scores", c_int, [c_void_p, c_int64, c_int32, c_void_p, c_int32, c_void_p,
                                     c_void_p]),
    ("rcb_topk_merge_shards", c_int, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int32,
                                      c_void_p, c_void_p, c_void_p]),
    ("rcb_peer_window_bytes", c_int64, [c_int32, c_int64]),
    ("rcb_peer_window_alloc", c_int, [c_int32, c_int64, POINTER(c_void_p)]),
    ("rcb_peer_window_free", c_int, [c_void_p]),
    ("rcb_peer_ipc_handle", c_int, [c_void_p, c_void_p]),
    ("rcb_peer_open", c_int, [c_void_p, POINTER(c_void_p)]),
    ("rcb_peer_close", c_int, [c_void_p]),
    ("rcb_peer_push", c_int, [POINTER(c_void_p), c_int32, c_int32, c_int64, c_void_p, c_void_p,
                              c_uint32, c_void_p]),
    ("rcb_peer_merge", c_int, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_uint32, c_uint64,
                               c_void_p, c_void_p, c_void_p, c_void_p]),
    ("rcb_peer_push_bytes", c_int, [POINTER(c_void_p), c_int32, c_int32, c_int64, c_void_p,
                                    c_int64, c_uint32, c_void_p]),
    ("rcb_peer_wait", c_int, [c_void_p, c_int32, c_int64, c_uint32, c_uint64, c_void_p, c_void_p]),
    ("rcb_peer_slot_offset", c_int64, [c_int32, c_int64, c_uint32]),
]

_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load the native library (once).  Raises RcbUnavailable if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RcbUnavailable(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - depends on the box
        raise RcbUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, restype, argtypes in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def check(code: int, what: str = "") -> None:
    if code != RCB_OK:
        msg = load().rcb_last_error().decode(errors="replace")
        raise RcbError(code, f"{what}: {msg}" if what else msg)


def i32_array(values) -> ctypes.Array:
    vals = list(values)
    return (c_int32 * max(1, len(vals)))(*vals)


def i64_array(values) -> ctypes.Array:
    vals = list(values)
    return (c_int64 * max(1, len(vals)))(*vals)


def stream_handle(stream) -> int:
    """cudaStream_t of a torch.cuda.Stream (or None -> legacy default stream)."""
    if stream is None:
        return 0
    return int(stream.cuda_stream)
