// block_pool.cpp — paged doc-KV block pool: HBM tier + pinned host tier.
//
// Executes the KV movements that the reference's knowledge tree only counts
// in tokens (ragsim tree.py:57-67 TierState, :296-333 load/reserve/release,
// :450-502 demote / free / drop).  Python (the reference's KnowledgeTree,
// unchanged) makes every decision; this pool owns memory and block ids.
//
// Allocation: lowest-free-block-first min-heaps in both tiers, so the block
// tables are a deterministic function of the tree's event stream
// (oracle/block_oracle.py restates the same rule).  Nodes are block-aligned
// (SURVEY H2): a node of n tokens owns ceil(n / block_tokens) blocks.
//
// Copies are batched per direction and issued in order on one copy stream
// (SURVEY H3): a block freed by a pending swap-out can only be rewritten by
// work that is ordered after the flush (swap-in on the same stream, or compute
// fenced with rcb_pool_fence_into, or per layer with rcb_pool_flush_layered +
// rcb_pool_fence_layer).
#include <algorithm>
#include <cstring>
#include <functional>
#include <queue>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "rcb_internal.h"

namespace {

struct MinHeap {
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> q;
  void init(int64_t n) {
    std::vector<int32_t> v(n);
    for (int64_t i = 0; i < n; ++i) v[i] = static_cast<int32_t>(i);
    q = decltype(q)(std::greater<int32_t>(), std::move(v));
  }
  int64_t size() const { return static_cast<int64_t>(q.size()); }
  void take(int32_t n, std::vector<int32_t>& out) {
    out.clear();
    out.reserve(n);
    for (int32_t i = 0; i < n; ++i) {
      out.push_back(q.top());
      q.pop();
    }
  }
  void give(const std::vector<int32_t>& blocks) {
    for (int32_t b : blocks) q.push(b);
  }
};

struct Node {
  int32_t tokens = 0;
  std::vector<int32_t> gpu;
  std::vector<int32_t> host;
};

struct Seg {
  int32_t tokens = 0;
  std::vector<int32_t> blocks;
  bool adopted = false;
};

struct Gen {
  std::vector<Seg> segs;
};

}  // namespace

struct rcb_pool {
  int64_t n_gpu = 0, n_host = 0;
  int32_t bt = 0, layers = 0, kv_heads = 0, head_dim = 0, elem_bytes = 0;
  int64_t block_bytes = 0;
  int32_t swap_mode = RCB_SWAP_STAGED;
  uint8_t* gpu_base = nullptr;
  bool own_gpu = false;
  uint8_t* host_base = nullptr;
  uint8_t* staging = nullptr;
  int64_t staging_blocks = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_done = nullptr, ev_dep = nullptr;
  MinHeap gpu_free, host_free;
  std::unordered_map<int64_t, Node> nodes;
  std::unordered_map<int64_t, Gen> gens;
  // pending copies, (gpu block, host block) pairs per direction.  Within a direction a
  // batch never names a block twice, so one launch / one DMA sequence is order-free (a
  // host block freed and reused inside a batch would otherwise race in the zero-copy
  // kernel).  Both directions may be pending at once: they are always issued swap-outs
  // first (per layer group when layered), which is the order every allowed overlap needs
  // (a swap-in writing a GPU block a pending swap-out still reads, or reading a host
  // block a pending swap-out writes).  Any other overlap flushes first (enqueue).
  std::vector<std::pair<int32_t, int32_t>> pend_out, pend_in;
  std::unordered_set<int32_t> out_gpu, out_host, in_gpu, in_host;
  int64_t stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // layer-pipelined swap-in (rcb_pool_flush_layered): one event per layer group
  // of the last layered H2D batch; invalidated by any later copy issue
  std::vector<cudaEvent_t> ev_layer;
  int32_t layered_groups = 0, group_layers = 0;

  int32_t nblocks(int32_t tokens) const { return (tokens + bt - 1) / bt; }
};

namespace {

using rcb::set_cuda_error;
using rcb::set_error;

int issue_runs(rcb_pool* p, const std::vector<std::pair<int32_t, int32_t>>& pr, size_t lo,
               size_t hi, bool to_host) {
  // staged: gather/scatter between pool blocks and staging slots [0, hi-lo), DMA
  // between staging and host runs.
  rcb::BlockPairs bp;
  const int n = static_cast<int>(hi - lo);
  for (int i = 0; i < n; ++i) {
    bp.src[i] = to_host ? pr[lo + i].first : i;
    bp.dst[i] = to_host ? i : pr[lo + i].first;
  }
  auto dma_runs = [&](bool d2h) -> int {
    size_t i = lo;
    while (i < hi) {
      size_t j = i + 1;
      while (j < hi && pr[j].second == pr[j - 1].second + 1) ++j;
      uint8_t* host = p->host_base + int64_t(pr[i].second) * p->block_bytes;
      uint8_t* stg = p->staging + int64_t(i - lo) * p->block_bytes;
      const size_t bytes = size_t(j - i) * p->block_bytes;
      cudaError_t e = d2h ? cudaMemcpyAsync(host, stg, bytes, cudaMemcpyDeviceToHost, p->stream)
                          : cudaMemcpyAsync(stg, host, bytes, cudaMemcpyHostToDevice, p->stream);
      if (e != cudaSuccess) return set_cuda_error(e, "pool staged memcpy");
      p->stats[7] += 1;
      i = j;
    }
    return RCB_OK;
  };
  if (to_host) {
    cudaError_t e = rcb::launch_block_copy_params(p->gpu_base, p->staging, p->block_bytes, bp, n,
                                                  p->stream);
    if (e != cudaSuccess) return set_cuda_error(e, "pool gather");
    p->stats[6] += 1;
    return dma_runs(true);
  }
  int rc = dma_runs(false);
  if (rc != RCB_OK) return rc;
  cudaError_t e =
      rcb::launch_block_copy_params(p->staging, p->gpu_base, p->block_bytes, bp, n, p->stream);
  if (e != cudaSuccess) return set_cuda_error(e, "pool scatter");
  p->stats[6] += 1;
  return RCB_OK;
}

void clear_pending(rcb_pool* p) {
  p->pend_out.clear();
  p->pend_in.clear();
  p->out_gpu.clear();
  p->out_host.clear();
  p->in_gpu.clear();
  p->in_host.clear();
}

bool any_pending(const rcb_pool* p) { return !p->pend_out.empty() || !p->pend_in.empty(); }

// one direction's batch, whole blocks, in the pool's swap mode
int issue_batch(rcb_pool* p, const std::vector<std::pair<int32_t, int32_t>>& pr, bool to_host) {
  if (pr.empty()) return RCB_OK;
  int rc = RCB_OK;
  if (p->swap_mode == RCB_SWAP_ZEROCOPY) {
    for (size_t lo = 0; lo < pr.size() && rc == RCB_OK; lo += rcb::kPairsPerLaunch) {
      const size_t hi = std::min(pr.size(), lo + rcb::kPairsPerLaunch);
      rcb::BlockPairs bp;
      for (size_t i = lo; i < hi; ++i) {
        bp.src[i - lo] = to_host ? pr[i].first : pr[i].second;
        bp.dst[i - lo] = to_host ? pr[i].second : pr[i].first;
      }
      cudaError_t e = to_host ? rcb::launch_block_copy_params(p->gpu_base, p->host_base,
                                                              p->block_bytes, bp, int(hi - lo),
                                                              p->stream)
                              : rcb::launch_block_copy_params(p->host_base, p->gpu_base,
                                                              p->block_bytes, bp, int(hi - lo),
                                                              p->stream);
      if (e != cudaSuccess) rc = set_cuda_error(e, "pool zero-copy swap");
      p->stats[6] += 1;
    }
  } else if (p->swap_mode == RCB_SWAP_DMA) {
    size_t i = 0;
    while (i < pr.size() && rc == RCB_OK) {
      size_t j = i + 1;
      while (j < pr.size() && pr[j].first == pr[j - 1].first + 1 &&
             pr[j].second == pr[j - 1].second + 1)
        ++j;
      uint8_t* g = p->gpu_base + int64_t(pr[i].first) * p->block_bytes;
      uint8_t* h = p->host_base + int64_t(pr[i].second) * p->block_bytes;
      const size_t bytes = size_t(j - i) * p->block_bytes;
      cudaError_t e = to_host ? cudaMemcpyAsync(h, g, bytes, cudaMemcpyDeviceToHost, p->stream)
                              : cudaMemcpyAsync(g, h, bytes, cudaMemcpyHostToDevice, p->stream);
      if (e != cudaSuccess) rc = set_cuda_error(e, "pool direct memcpy");
      p->stats[7] += 1;
      i = j;
    }
  } else {
    const size_t chunk =
        static_cast<size_t>(std::min<int64_t>(p->staging_blocks, rcb::kPairsPerLaunch));
    for (size_t lo = 0; lo < pr.size() && rc == RCB_OK; lo += chunk)
      rc = issue_runs(p, pr, lo, std::min(pr.size(), lo + chunk), to_host);
  }
  return rc;
}

int flush(rcb_pool* p) {
  const int64_t out_bytes = static_cast<int64_t>(p->pend_out.size()) * p->block_bytes;
  const int64_t in_bytes = static_cast<int64_t>(p->pend_in.size()) * p->block_bytes;
  int rc = RCB_OK;
  if (p->swap_mode != RCB_POOL_ACCOUNTING && any_pending(p)) {
    p->layered_groups = 0;  // later copies are not covered by the per-layer events
    rc = issue_batch(p, p->pend_out, true);  // swap-outs first (see pend_out)
    if (rc == RCB_OK) rc = issue_batch(p, p->pend_in, false);
  }
  p->stats[2] += out_bytes;
  p->stats[3] += in_bytes;
  clear_pending(p);
  return rc;
}

// dir 1: swap-out (GPU g -> host h), 2: swap-in (host h -> GPU g)
int enqueue(rcb_pool* p, int dir, const std::vector<int32_t>& g, const std::vector<int32_t>& h) {
  bool conflict = false;
  for (size_t i = 0; i < g.size() && !conflict; ++i) {
    if (dir == 1)  // must follow every pending copy that touches its blocks: flush first
      conflict = p->out_gpu.count(g[i]) || p->out_host.count(h[i]) || p->in_gpu.count(g[i]) ||
                 p->in_host.count(h[i]);
    else  // after a pending swap-out on the same block is fine: swap-outs issue first
      conflict = p->in_gpu.count(g[i]) || p->in_host.count(h[i]);
  }
  if (conflict) {
    int rc = flush(p);
    if (rc != RCB_OK) return rc;
  }
  auto& list = dir == 1 ? p->pend_out : p->pend_in;
  auto& sg = dir == 1 ? p->out_gpu : p->in_gpu;
  auto& sh = dir == 1 ? p->out_host : p->in_host;
  for (size_t i = 0; i < g.size(); ++i) {
    list.emplace_back(g[i], h[i]);
    sg.insert(g[i]);
    sh.insert(h[i]);
  }
  return RCB_OK;
}

// Layer-pipelined swaps: the pending batches are issued as G groups of
// `lpg` layers.  Within a block the layer slices are contiguous ([L][2][H_kv][B][d_h]),
// so group g of a run of consecutive (gpu, host) block pairs is ONE strided DMA
// (cudaMemcpy2DAsync: width = lpg layer slices, pitch = block_bytes, height = run
// length), and the copy engines do the scatter (no SMs taken from the prefill).  Per
// group the swap-out slices go first, then the swap-in slices (the order of pend_out);
// event g is recorded after group g.  A prefill's layer l waits only for its group
// (rcb_pool_fence_layer): its K/V write may then reuse blocks whose layer-l slices a
// swap-out has already read, and its attention reads swapped-in layer-l slices.
int flush_layered(rcb_pool* p, int32_t lpg) {
  const int32_t groups = (p->layers + lpg - 1) / lpg;
  while (static_cast<int32_t>(p->ev_layer.size()) < groups) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return set_cuda_error(e, "pool layer event");
    p->ev_layer.push_back(ev);
  }
  using Runs = std::vector<std::pair<size_t, size_t>>;  // [i, j): consecutive gpu and host blocks
  auto runs_of = [](const std::vector<std::pair<int32_t, int32_t>>& pr) {
    Runs runs;
    for (size_t i = 0; i < pr.size();) {
      size_t j = i + 1;
      while (j < pr.size() && pr[j].first == pr[j - 1].first + 1 &&
             pr[j].second == pr[j - 1].second + 1)
        ++j;
      runs.emplace_back(i, j);
      i = j;
    }
    return runs;
  };
  const Runs runs_out = runs_of(p->pend_out), runs_in = runs_of(p->pend_in);
  const int64_t layer_bytes = p->block_bytes / p->layers;
  for (int32_t g = 0; g < groups; ++g) {
    const int32_t l0 = g * lpg, l1 = std::min(p->layers, l0 + lpg);
    const int64_t off = int64_t(l0) * layer_bytes, width = int64_t(l1 - l0) * layer_bytes;
    for (int d = 0; d < 2; ++d) {
      const bool to_host = d == 0;
      const auto& pr = to_host ? p->pend_out : p->pend_in;
      for (const auto& r : to_host ? runs_out : runs_in) {
        uint8_t* gp = p->gpu_base + int64_t(pr[r.first].first) * p->block_bytes + off;
        uint8_t* hp = p->host_base + int64_t(pr[r.first].second) * p->block_bytes + off;
        cudaError_t e =
            to_host ? cudaMemcpy2DAsync(hp, p->block_bytes, gp, p->block_bytes, width,
                                        r.second - r.first, cudaMemcpyDeviceToHost, p->stream)
                    : cudaMemcpy2DAsync(gp, p->block_bytes, hp, p->block_bytes, width,
                                        r.second - r.first, cudaMemcpyHostToDevice, p->stream);
        if (e != cudaSuccess) return set_cuda_error(e, "pool layered memcpy");
        p->stats[7] += 1;
      }
    }
    cudaError_t e = cudaEventRecord(p->ev_layer[g], p->stream);
    if (e != cudaSuccess) return set_cuda_error(e, "pool layer event record");
  }
  p->stats[2] += static_cast<int64_t>(p->pend_out.size()) * p->block_bytes;
  p->stats[3] += static_cast<int64_t>(p->pend_in.size()) * p->block_bytes;
  clear_pending(p);
  p->layered_groups = groups;
  p->group_layers = lpg;
  return RCB_OK;
}

}  // namespace

extern "C" {

int rcb_pool_create(int64_t num_gpu_blocks, int64_t num_host_blocks, int32_t block_tokens,
                    int32_t n_layers, int32_t n_kv_heads, int32_t head_dim, int32_t elem_bytes,
                    int32_t swap_mode, void* gpu_base, void* copy_stream, rcb_pool** out) {
  if (out == nullptr) return set_error(RCB_ERR_ARG, "null out");
  *out = nullptr;
  if (num_gpu_blocks <= 0 || num_host_blocks < 0 || block_tokens <= 0 || n_layers <= 0 ||
      n_kv_heads <= 0 || head_dim <= 0 || elem_bytes <= 0 || num_gpu_blocks >= (1ll << 31) ||
      num_host_blocks >= (1ll << 31))
    return set_error(RCB_ERR_ARG, "bad pool geometry");
  if (swap_mode < RCB_SWAP_STAGED || swap_mode > RCB_POOL_ACCOUNTING)
    return set_error(RCB_ERR_ARG, "bad swap mode");
  rcb_pool* p = new rcb_pool();
  p->n_gpu = num_gpu_blocks;
  p->n_host = num_host_blocks;
  p->bt = block_tokens;
  p->layers = n_layers;
  p->kv_heads = n_kv_heads;
  p->head_dim = head_dim;
  p->elem_bytes = elem_bytes;
  p->block_bytes = int64_t(n_layers) * 2 * n_kv_heads * block_tokens * head_dim * elem_bytes;
  if (p->block_bytes % 16 != 0) {
    delete p;
    return set_error(RCB_ERR_ARG, "block bytes must be a multiple of 16");
  }
  p->swap_mode = swap_mode;
  if (swap_mode == RCB_POOL_ACCOUNTING) {
    p->gpu_free.init(num_gpu_blocks);
    p->host_free.init(num_host_blocks);
    *out = p;
    return RCB_OK;
  }
  cudaError_t e;
  if (gpu_base != nullptr) {
    p->gpu_base = static_cast<uint8_t*>(gpu_base);
  } else {
    e = cudaMalloc(&p->gpu_base, num_gpu_blocks * p->block_bytes);
    if (e != cudaSuccess) {
      delete p;
      return set_cuda_error(e, "pool cudaMalloc");
    }
    p->own_gpu = true;
    // attention never reads uninitialised (possibly NaN) bytes from masked slots
    e = cudaMemset(p->gpu_base, 0, num_gpu_blocks * p->block_bytes);
    if (e != cudaSuccess) {
      cudaFree(p->gpu_base);
      delete p;
      return set_cuda_error(e, "pool cudaMemset");
    }
  }
  if (num_host_blocks > 0) {
    e = cudaHostAlloc(&p->host_base, num_host_blocks * p->block_bytes,
                      cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) {
      if (p->own_gpu) cudaFree(p->gpu_base);
      delete p;
      return set_cuda_error(e, "pool cudaHostAlloc");
    }
  }
  const int64_t staging_cap = std::max<int64_t>(1, (int64_t(256) << 20) / p->block_bytes);
  p->staging_blocks = std::min<int64_t>(staging_cap, std::max<int64_t>(1, num_host_blocks));
  e = cudaMalloc(&p->staging, p->staging_blocks * p->block_bytes);
  if (e == cudaSuccess && copy_stream == nullptr) {
    e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
    p->own_stream = true;
  } else {
    p->stream = static_cast<cudaStream_t>(copy_stream);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_dep, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    rcb_pool_destroy(p);
    return set_cuda_error(e, "pool stream/staging");
  }
  p->gpu_free.init(num_gpu_blocks);
  p->host_free.init(num_host_blocks);
  *out = p;
  return RCB_OK;
}

int rcb_pool_destroy(rcb_pool* p) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (p->stream) cudaStreamSynchronize(p->stream);
  if (p->ev_done) cudaEventDestroy(p->ev_done);
  if (p->ev_dep) cudaEventDestroy(p->ev_dep);
  for (cudaEvent_t ev : p->ev_layer) cudaEventDestroy(ev);
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  if (p->staging) cudaFree(p->staging);
  if (p->host_base) cudaFreeHost(p->host_base);
  if (p->own_gpu && p->gpu_base) cudaFree(p->gpu_base);
  delete p;
  return RCB_OK;
}

int rcb_pool_info(rcb_pool* p, int64_t* out) {
  if (p == nullptr || out == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  out[0] = reinterpret_cast<int64_t>(p->gpu_base);
  out[1] = reinterpret_cast<int64_t>(p->host_base);
  out[2] = p->block_bytes;
  out[3] = p->gpu_free.size();
  out[4] = p->host_free.size();
  out[5] = p->n_gpu;
  out[6] = p->n_host;
  return RCB_OK;
}

int rcb_pool_stats(rcb_pool* p, int64_t* out) {
  if (p == nullptr || out == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  std::memcpy(out, p->stats, sizeof(p->stats));
  return RCB_OK;
}

int rcb_pool_set_swap_mode(rcb_pool* p, int32_t mode) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (mode < RCB_SWAP_STAGED || mode > RCB_SWAP_DMA || p->swap_mode == RCB_POOL_ACCOUNTING)
    return set_error(RCB_ERR_ARG, "bad mode");
  int rc = flush(p);
  p->swap_mode = mode;
  return rc;
}

int rcb_node_alloc_gpu(rcb_pool* p, int64_t key, int32_t n_tokens) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (n_tokens <= 0) return set_error(RCB_ERR_ARG, "node needs positive tokens");
  auto it = p->nodes.find(key);
  if (it != p->nodes.end() && !it->second.gpu.empty())
    return set_error(RCB_ERR_BAD_HANDLE, "node already GPU-resident");
  const int32_t nb = p->nblocks(n_tokens);
  if (p->gpu_free.size() < nb) return set_error(RCB_ERR_NO_BLOCKS, "out of GPU blocks");
  Node& n = p->nodes[key];
  n.tokens = n_tokens;
  p->gpu_free.take(nb, n.gpu);
  return RCB_OK;
}

int rcb_node_free_gpu(rcb_pool* p, int64_t key) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  auto it = p->nodes.find(key);
  if (it == p->nodes.end() || it->second.gpu.empty())
    return set_error(RCB_ERR_BAD_HANDLE, "node not GPU-resident");
  p->gpu_free.give(it->second.gpu);
  it->second.gpu.clear();
  if (it->second.host.empty()) p->nodes.erase(it);
  return RCB_OK;
}

int rcb_node_free_host(rcb_pool* p, int64_t key) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  auto it = p->nodes.find(key);
  if (it == p->nodes.end() || it->second.host.empty())
    return set_error(RCB_ERR_BAD_HANDLE, "node has no host copy");
  p->host_free.give(it->second.host);
  it->second.host.clear();
  if (it->second.gpu.empty()) p->nodes.erase(it);
  return RCB_OK;
}

// a key repeated in one batch would pass the per-key validation twice and then leak /
// overwrite its blocks in the mutation loop: rejected before any state changes
static bool has_duplicate(const int64_t* keys, int32_t n) {
  std::unordered_set<int64_t> seen;
  for (int32_t i = 0; i < n; ++i)
    if (!seen.insert(keys[i]).second) return true;
  return false;
}

int rcb_node_swap_out(rcb_pool* p, const int64_t* keys, int32_t n) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (has_duplicate(keys, n)) return set_error(RCB_ERR_ARG, "swap-out: duplicate node key");
  int64_t need = 0;
  for (int32_t i = 0; i < n; ++i) {
    auto it = p->nodes.find(keys[i]);
    if (it == p->nodes.end() || it->second.gpu.empty() || !it->second.host.empty())
      return set_error(RCB_ERR_BAD_HANDLE, "swap-out needs a GPU node without host copy");
    need += p->nblocks(it->second.tokens);
  }
  if (p->host_free.size() < need) return set_error(RCB_ERR_NO_BLOCKS, "out of host blocks");
  for (int32_t i = 0; i < n; ++i) {
    Node& nd = p->nodes[keys[i]];
    p->host_free.take(p->nblocks(nd.tokens), nd.host);
    int rc = enqueue(p, 1, nd.gpu, nd.host);
    if (rc != RCB_OK) return rc;
    p->stats[0] += static_cast<int64_t>(nd.gpu.size());
    p->gpu_free.give(nd.gpu);
    nd.gpu.clear();
  }
  p->stats[4] += 1;
  return RCB_OK;
}

int rcb_node_swap_in(rcb_pool* p, const int64_t* keys, int32_t n) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (has_duplicate(keys, n)) return set_error(RCB_ERR_ARG, "swap-in: duplicate node key");
  int64_t need = 0;
  for (int32_t i = 0; i < n; ++i) {
    auto it = p->nodes.find(keys[i]);
    if (it == p->nodes.end() || it->second.host.empty() || !it->second.gpu.empty())
      return set_error(RCB_ERR_BAD_HANDLE, "swap-in needs a host-only node");
    need += p->nblocks(it->second.tokens);
  }
  if (p->gpu_free.size() < need) return set_error(RCB_ERR_NO_BLOCKS, "out of GPU blocks");
  for (int32_t i = 0; i < n; ++i) {
    Node& nd = p->nodes[keys[i]];
    p->gpu_free.take(p->nblocks(nd.tokens), nd.gpu);
    int rc = enqueue(p, 2, nd.gpu, nd.host);
    if (rc != RCB_OK) return rc;
    p->stats[1] += static_cast<int64_t>(nd.gpu.size());
  }
  p->stats[5] += 1;
  return RCB_OK;
}

int rcb_gen_reserve(rcb_pool* p, int64_t gen_key, const int32_t* seg_tokens, int32_t nseg) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (p->gens.count(gen_key)) return set_error(RCB_ERR_BAD_HANDLE, "generation already reserved");
  int64_t need = 0;
  for (int32_t i = 0; i < nseg; ++i) {
    if (seg_tokens[i] <= 0) return set_error(RCB_ERR_ARG, "segment needs positive tokens");
    need += p->nblocks(seg_tokens[i]);
  }
  if (p->gpu_free.size() < need) return set_error(RCB_ERR_NO_BLOCKS, "out of GPU blocks");
  Gen& g = p->gens[gen_key];
  g.segs.resize(nseg);
  for (int32_t i = 0; i < nseg; ++i) {
    g.segs[i].tokens = seg_tokens[i];
    p->gpu_free.take(p->nblocks(seg_tokens[i]), g.segs[i].blocks);
  }
  return RCB_OK;
}

int rcb_node_adopt(rcb_pool* p, int64_t key, int64_t gen_key, int32_t seg_idx) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  auto git = p->gens.find(gen_key);
  if (git == p->gens.end() || seg_idx < 0 || seg_idx >= (int32_t)git->second.segs.size())
    return set_error(RCB_ERR_BAD_HANDLE, "unknown generation segment");
  Seg& s = git->second.segs[seg_idx];
  if (s.adopted) return set_error(RCB_ERR_BAD_HANDLE, "segment already adopted");
  auto it = p->nodes.find(key);
  if (it != p->nodes.end() && !it->second.gpu.empty())
    return set_error(RCB_ERR_BAD_HANDLE, "adopting node already GPU-resident");
  Node& nd = p->nodes[key];
  nd.tokens = s.tokens;
  nd.gpu = std::move(s.blocks);
  s.blocks.clear();
  s.adopted = true;
  return RCB_OK;
}

int rcb_gen_free_segment(rcb_pool* p, int64_t gen_key, int32_t seg_idx) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  auto git = p->gens.find(gen_key);
  if (git == p->gens.end() || seg_idx < 0 || seg_idx >= (int32_t)git->second.segs.size())
    return set_error(RCB_ERR_BAD_HANDLE, "unknown generation segment");
  Seg& s = git->second.segs[seg_idx];
  if (s.adopted) return set_error(RCB_ERR_BAD_HANDLE, "segment already adopted or freed");
  p->gpu_free.give(s.blocks);
  s.blocks.clear();
  s.adopted = true;  // consumed: no longer part of the generation
  return RCB_OK;
}

int rcb_gen_release(rcb_pool* p, int64_t gen_key) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  auto git = p->gens.find(gen_key);
  if (git == p->gens.end()) return set_error(RCB_ERR_BAD_HANDLE, "unknown generation");
  for (Seg& s : git->second.segs)
    if (!s.adopted) p->gpu_free.give(s.blocks);
  p->gens.erase(git);
  return RCB_OK;
}

static int copy_out(const std::vector<int32_t>& v, int32_t* out, int32_t cap, int32_t* n_out) {
  if (n_out) *n_out = static_cast<int32_t>(v.size());
  if (static_cast<int32_t>(v.size()) > cap) return set_error(RCB_ERR_ARG, "output capacity too small");
  if (out && !v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(int32_t));
  return RCB_OK;
}

int rcb_node_blocks(rcb_pool* p, int64_t key, int32_t tier, int32_t* out, int32_t cap,
                    int32_t* n_out) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  auto it = p->nodes.find(key);
  static const std::vector<int32_t> empty;
  if (it == p->nodes.end()) return copy_out(empty, out, cap, n_out);
  return copy_out(tier == RCB_TIER_GPU ? it->second.gpu : it->second.host, out, cap, n_out);
}

int rcb_gen_blocks(rcb_pool* p, int64_t gen_key, int32_t seg_idx, int32_t* out, int32_t cap,
                   int32_t* n_out) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  auto git = p->gens.find(gen_key);
  if (git == p->gens.end() || seg_idx < 0 || seg_idx >= (int32_t)git->second.segs.size())
    return set_error(RCB_ERR_BAD_HANDLE, "unknown generation segment");
  return copy_out(git->second.segs[seg_idx].blocks, out, cap, n_out);
}

int rcb_block_table(rcb_pool* p, const int64_t* node_keys, int32_t n_nodes, int64_t gen_key,
                    int32_t* blocks_out, int32_t* valid_out, int32_t cap, int32_t* n_out) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  int32_t n = 0;
  auto push = [&](const std::vector<int32_t>& blocks, int32_t tokens) -> int {
    for (size_t i = 0; i < blocks.size(); ++i) {
      if (n >= cap) return set_error(RCB_ERR_ARG, "block table capacity too small");
      blocks_out[n] = blocks[i];
      valid_out[n] = (i + 1 < blocks.size()) ? p->bt : tokens - int32_t(i) * p->bt;
      ++n;
    }
    return RCB_OK;
  };
  for (int32_t i = 0; i < n_nodes; ++i) {
    auto it = p->nodes.find(node_keys[i]);
    if (it == p->nodes.end() || it->second.gpu.empty())
      return set_error(RCB_ERR_BAD_HANDLE, "block table node not GPU-resident");
    int rc = push(it->second.gpu, it->second.tokens);
    if (rc != RCB_OK) return rc;
  }
  if (gen_key >= 0) {
    auto git = p->gens.find(gen_key);
    if (git == p->gens.end()) return set_error(RCB_ERR_BAD_HANDLE, "unknown generation");
    for (const Seg& s : git->second.segs) {
      if (s.adopted) return set_error(RCB_ERR_BAD_HANDLE, "generation segment already adopted");
      int rc = push(s.blocks, s.tokens);
      if (rc != RCB_OK) return rc;
    }
  }
  if (n_out) *n_out = n;
  return RCB_OK;
}

int rcb_pool_flush(rcb_pool* p) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  return flush(p);
}

int rcb_pool_fence_into(rcb_pool* p, void* stream) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  int rc = flush(p);
  if (rc != RCB_OK || p->swap_mode == RCB_POOL_ACCOUNTING) return rc;
  cudaError_t e = cudaEventRecord(p->ev_done, p->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), p->ev_done, 0);
  if (e != cudaSuccess) return set_cuda_error(e, "pool fence_into");
  return RCB_OK;
}

int rcb_pool_wait_for(rcb_pool* p, void* stream) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (p->swap_mode == RCB_POOL_ACCOUNTING) return RCB_OK;
  cudaError_t e = cudaEventRecord(p->ev_dep, static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->stream, p->ev_dep, 0);
  if (e != cudaSuccess) return set_cuda_error(e, "pool wait_for");
  return RCB_OK;
}

int rcb_pool_flush_layered(rcb_pool* p, int32_t layers_per_group) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (layers_per_group <= 0) return set_error(RCB_ERR_ARG, "layers_per_group must be positive");
  if (p->swap_mode == RCB_POOL_ACCOUNTING || !any_pending(p)) return flush(p);
  return flush_layered(p, std::min(layers_per_group, p->layers));
}

int rcb_pool_fence_layer(rcb_pool* p, int32_t layer, void* stream) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (layer < 0 || layer >= p->layers) return set_error(RCB_ERR_ARG, "layer out of range");
  if (p->swap_mode == RCB_POOL_ACCOUNTING) return RCB_OK;
  if (any_pending(p) || p->layered_groups == 0)
    return rcb_pool_fence_into(p, stream);  // no layered batch outstanding: full fence
  const int32_t g = std::min(layer / p->group_layers, p->layered_groups - 1);
  cudaError_t e = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), p->ev_layer[g], 0);
  if (e != cudaSuccess) return set_cuda_error(e, "pool fence_layer");
  return RCB_OK;
}

int rcb_pool_drain(rcb_pool* p) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  if (p->swap_mode == RCB_POOL_ACCOUNTING) return RCB_OK;
  if (!p->pend_out.empty()) {  // a pending swap-out batch is issued and drained too; a
    // pending swap-in batch stays pending (it is issued later on the same stream, so it
    // still follows the swap-outs)
    p->layered_groups = 0;
    int rc = issue_batch(p, p->pend_out, true);
    p->stats[2] += static_cast<int64_t>(p->pend_out.size()) * p->block_bytes;
    p->pend_out.clear();
    p->out_gpu.clear();
    p->out_host.clear();
    if (rc != RCB_OK) return rc;
  }
  cudaError_t e = cudaStreamSynchronize(p->stream);
  if (e != cudaSuccess) return set_cuda_error(e, "pool drain");
  return RCB_OK;
}

int rcb_pool_sync(rcb_pool* p) {
  if (p == nullptr) return set_error(RCB_ERR_BAD_HANDLE, "null pool");
  int rc = flush(p);
  if (rc != RCB_OK || p->swap_mode == RCB_POOL_ACCOUNTING) return rc;
  cudaError_t e = cudaStreamSynchronize(p->stream);
  if (e != cudaSuccess) return set_cuda_error(e, "pool sync");
  return RCB_OK;
}

}  // extern "C"
