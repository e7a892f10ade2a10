// peer.cu — the sharded retrieval's list exchange over peer memory.
//
// SURVEY.md §8e / simulator.py:228: with the corpus sharded across the GPUs of a box,
// every rank scans its shard for all ranks' queries and the per-shard staged top-k lists
// are merged.  Instead of two NCCL all-gathers (ids, scores) followed by the merge, each
// rank writes its lists straight into every peer's exchange window (CUDA IPC mapping:
// NVLink P2P stores on a multi-GPU box) and publishes an epoch flag with a system-scope
// release; each rank's merge waits for all flags (acquire) and reads its own window.
//
// Window (one cudaMalloc per rank, exported with cudaIpcGetMemHandle):
//   ids    int64 [2 parity][n_ranks][n_entries]
//   scores f32   [2 parity][n_ranks][n_entries]
//   flags  u32   [n_ranks]       (last epoch each sender published)
// n_entries = n_queries * n_stages * k, the shard-merge input layout.  Epoch e uses parity
// e & 1: a rank can only push epoch e + 1 after the step's query all-gather, i.e. after
// every rank issued its epoch-e merge, so a slot is never overwritten while being read.
#include <climits>
#include <cstring>

#include "rcb_internal.h"

namespace rcb {
namespace peer {

constexpr int kMaxRanks = 8;

struct Windows {
  uint8_t* w[kMaxRanks];
};

struct Layout {
  int64_t ids, scores, flags, bytes;
};

__host__ __device__ inline Layout layout(int n_ranks, int64_t n_entries) {
  Layout l;
  l.ids = 0;
  l.scores = l.ids + 2 * int64_t(n_ranks) * n_entries * 8;
  l.flags = l.scores + ((2 * int64_t(n_ranks) * n_entries * 4 + 127) / 128) * 128;
  l.bytes = l.flags + 128;
  return l;
}

// grid = n_ranks (one CTA per destination), 256 threads: copy this rank's lists into slot
// [parity][rank] of destination p, then publish the epoch in p's flags[rank]
__global__ void __launch_bounds__(256)
    push_kernel(Windows win, int n_ranks, int rank, int64_t n_entries,
                const long long* __restrict__ ids, const float* __restrict__ scores,
                unsigned epoch) {
  const int p = blockIdx.x;
  const Layout l = layout(n_ranks, n_entries);
  uint8_t* w = win.w[p];
  const int64_t slot = (int64_t(epoch & 1) * n_ranks + rank) * n_entries;
  long long* di = reinterpret_cast<long long*>(w + l.ids) + slot;
  float* ds = reinterpret_cast<float*>(w + l.scores) + slot;
  for (int64_t i = threadIdx.x; i < n_entries; i += blockDim.x) {
    di[i] = ids[i];
    ds[i] = scores[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned* f = reinterpret_cast<unsigned*>(w + l.flags) + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
}

// generic form: copy `bytes` (a multiple of 8) into the ids region slot [parity][rank] of
// destination p, then publish the epoch (the query exchange uses it for bf16 rows)
__global__ void __launch_bounds__(256)
    push_bytes_kernel(Windows win, int n_ranks, int rank, int64_t n_entries,
                      const long long* __restrict__ src, int64_t words, unsigned epoch) {
  const int p = blockIdx.x;
  const Layout l = layout(n_ranks, n_entries);
  uint8_t* w = win.w[p];
  long long* d = reinterpret_cast<long long*>(w + l.ids) + (int64_t(epoch & 1) * n_ranks + rank) * n_entries;
  for (int64_t i = threadIdx.x; i < words; i += blockDim.x) d[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned* f = reinterpret_cast<unsigned*>(w + l.flags) + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
}

// one thread: wait (acquire) until every sender published `epoch`; bounded, so a missing
// peer sets *timed_out instead of hanging the device
__global__ void wait_kernel(const uint8_t* __restrict__ window, int n_ranks, int64_t n_entries,
                            unsigned epoch, unsigned long long timeout_ns, int* timed_out) {
  const Layout l = layout(n_ranks, n_entries);
  const unsigned* f = reinterpret_cast<const unsigned*>(window + l.flags);
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < n_ranks; ++r) {
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f + r) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        *timed_out = 1;
        return;
      }
      __nanosleep(200);
    }
  }
}

}  // namespace peer
}  // namespace rcb

using rcb::set_cuda_error;
using rcb::set_error;

extern "C" {

int64_t rcb_peer_window_bytes(int32_t n_ranks, int64_t n_entries) {
  if (n_ranks < 1 || n_ranks > rcb::peer::kMaxRanks || n_entries < 1) return -1;
  return rcb::peer::layout(n_ranks, n_entries).bytes;
}

int rcb_peer_window_alloc(int32_t n_ranks, int64_t n_entries, void** window_out) {
  const int64_t bytes = rcb_peer_window_bytes(n_ranks, n_entries);
  if (bytes < 0 || window_out == nullptr) return set_error(RCB_ERR_ARG, "bad peer window shape");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);  // its own allocation: exportable with cudaIpc
  if (e != cudaSuccess) return set_cuda_error(e, "peer window alloc");
  e = cudaMemset(p, 0, bytes);  // flags start at epoch 0; pushes begin at epoch 1
  if (e != cudaSuccess) return set_cuda_error(e, "peer window clear");
  *window_out = p;
  return RCB_OK;
}

int rcb_peer_window_free(void* window) {
  cudaError_t e = cudaFree(window);
  return e == cudaSuccess ? RCB_OK : set_cuda_error(e, "peer window free");
}

int rcb_peer_ipc_handle(void* window, void* handle_out) {
  if (handle_out == nullptr) return set_error(RCB_ERR_ARG, "null handle");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, window);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == RCB_PEER_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  return RCB_OK;
}

int rcb_peer_open(const void* handle, void** window_out) {
  if (handle == nullptr || window_out == nullptr) return set_error(RCB_ERR_ARG, "null handle");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaIpcOpenMemHandle");
  *window_out = p;
  return RCB_OK;
}

int rcb_peer_close(void* window) {
  cudaError_t e = cudaIpcCloseMemHandle(window);
  return e == cudaSuccess ? RCB_OK : set_cuda_error(e, "cudaIpcCloseMemHandle");
}

int rcb_peer_push(void* const* windows, int32_t n_ranks, int32_t rank, int64_t n_entries,
                  const int64_t* ids_dev, const float* scores_dev, uint32_t epoch,
                  void* stream) {
  if (n_ranks < 1 || n_ranks > rcb::peer::kMaxRanks || rank < 0 || rank >= n_ranks ||
      n_entries < 1 || windows == nullptr || epoch == 0)
    return set_error(RCB_ERR_ARG, "bad peer push arguments");
  rcb::peer::Windows w{};
  for (int r = 0; r < n_ranks; ++r) {
    if (windows[r] == nullptr) return set_error(RCB_ERR_ARG, "missing peer window");
    w.w[r] = static_cast<uint8_t*>(windows[r]);
  }
  rcb::peer::push_kernel<<<n_ranks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w, n_ranks, rank, n_entries, reinterpret_cast<const long long*>(ids_dev), scores_dev,
      epoch);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RCB_OK : set_cuda_error(e, "peer push launch");
}

int rcb_peer_merge(const void* window, int32_t n_ranks, int32_t n_queries, int32_t n_stages,
                   int32_t k, uint32_t epoch, uint64_t timeout_ns, int32_t* timed_out_dev,
                   int64_t* ids_out_dev, float* scores_out_dev, void* stream) {
  const int64_t n_entries = int64_t(n_queries) * n_stages * k;
  if (rcb_peer_window_bytes(n_ranks, n_entries) < 0 || epoch == 0 || timed_out_dev == nullptr)
    return set_error(RCB_ERR_ARG, "bad peer merge arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint8_t* w = static_cast<const uint8_t*>(window);
  rcb::peer::wait_kernel<<<1, 1, 0, st>>>(w, n_ranks, n_entries, epoch, timeout_ns, timed_out_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "peer wait launch");
  const rcb::peer::Layout l = rcb::peer::layout(n_ranks, n_entries);
  const int64_t slot = int64_t(epoch & 1) * n_ranks * n_entries;
  return rcb_topk_merge_shards(reinterpret_cast<const int64_t*>(w + l.ids) + slot,
                               reinterpret_cast<const float*>(w + l.scores) + slot, n_ranks,
                               n_queries, n_stages, k, ids_out_dev, scores_out_dev, stream);
}

int rcb_peer_push_bytes(void* const* windows, int32_t n_ranks, int32_t rank, int64_t n_entries,
                        const void* src_dev, int64_t bytes, uint32_t epoch, void* stream) {
  if (n_ranks < 1 || n_ranks > rcb::peer::kMaxRanks || rank < 0 || rank >= n_ranks ||
      n_entries < 1 || windows == nullptr || epoch == 0 || bytes < 8 || bytes % 8 != 0 ||
      bytes > n_entries * 8 || reinterpret_cast<uintptr_t>(src_dev) % 8 != 0)
    return set_error(RCB_ERR_ARG, "bad peer byte push arguments");
  rcb::peer::Windows w{};
  for (int r = 0; r < n_ranks; ++r) {
    if (windows[r] == nullptr) return set_error(RCB_ERR_ARG, "missing peer window");
    w.w[r] = static_cast<uint8_t*>(windows[r]);
  }
  rcb::peer::push_bytes_kernel<<<n_ranks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w, n_ranks, rank, n_entries, static_cast<const long long*>(src_dev), bytes / 8, epoch);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RCB_OK : set_cuda_error(e, "peer byte push launch");
}

int rcb_peer_wait(const void* window, int32_t n_ranks, int64_t n_entries, uint32_t epoch,
                  uint64_t timeout_ns, int32_t* timed_out_dev, void* stream) {
  if (rcb_peer_window_bytes(n_ranks, n_entries) < 0 || epoch == 0 || timed_out_dev == nullptr)
    return set_error(RCB_ERR_ARG, "bad peer wait arguments");
  rcb::peer::wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(window), n_ranks, n_entries, epoch, timeout_ns, timed_out_dev);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RCB_OK : set_cuda_error(e, "peer wait launch");
}

int64_t rcb_peer_slot_offset(int32_t n_ranks, int64_t n_entries, uint32_t epoch) {
  if (rcb_peer_window_bytes(n_ranks, n_entries) < 0) return -1;
  return rcb::peer::layout(n_ranks, n_entries).ids + int64_t(epoch & 1) * n_ranks * n_entries * 8;
}

}  // extern "C"
