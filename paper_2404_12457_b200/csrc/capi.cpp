// capi.cpp — C-ABI glue: error reporting, TMA descriptor encoding, the
// prefill entry point and its host-side work planner.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cudaTypedefs.h>
#include <string>
#include <vector>

#include "rcb_internal.h"

namespace rcb {

namespace {
thread_local std::string g_last_error;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
}  // namespace

int set_error(int code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}

int set_cuda_error(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return RCB_ERR_CUDA;
}

int encode_tma_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                    const uint64_t* strides, const uint32_t* box) {
  if (g_encode == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || fn == nullptr)
      return set_error(RCB_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t gdim[5];
  cuuint64_t gstr[4];
  cuuint32_t bx[5];
  cuuint32_t es[5];
  for (int i = 0; i < rank; ++i) {
    gdim[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
  }
  for (int i = 0; i + 1 < rank; ++i) gstr[i] = strides[i];
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), gdim,
                        gstr, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (CUresult %d, rank %d)",
                  (int)r, rank);
    return set_error(RCB_ERR_ARG, buf);
  }
  return RCB_OK;
}

}  // namespace rcb

extern "C" {

const char* rcb_last_error(void) { return rcb::g_last_error.c_str(); }

int rcb_version(void) { return 1; }

int rcb_prefix_prefill(const void* q, int64_t q_row_stride, void* o, int32_t total_q_tokens,
                       int32_t n_q_heads, const void* kv_pool, int64_t num_pool_blocks,
                       int32_t block_tokens, int32_t n_layers, int32_t n_kv_heads,
                       int32_t head_dim, int32_t layer, const int32_t* req_meta_dev,
                       const int32_t* blk_ids_dev, const int32_t* blk_valid_dev,
                       const int32_t* blk_pos_dev, const int32_t* work_dev, int32_t n_work,
                       float softmax_scale, const void* rope_table_dev, int32_t work_flags,
                       void* part_ws_dev, int32_t n_part_slots, const int32_t* combine_dev,
                       int32_t n_combine, void* stream) {
  if (block_tokens != 16 && block_tokens != 32 && block_tokens != 64 && block_tokens != 128)
    return rcb::set_error(RCB_ERR_ARG, "block_tokens must be 16, 32, 64 or 128");
  return rcb::prefix_prefill(q, q_row_stride, o, total_q_tokens, n_q_heads, kv_pool,
                             num_pool_blocks, block_tokens, n_layers, n_kv_heads, head_dim, layer,
                             req_meta_dev, blk_ids_dev, blk_valid_dev, blk_pos_dev, work_dev,
                             n_work, softmax_scale, rope_table_dev, work_flags, part_ws_dev,
                             n_part_slots, combine_dev, n_combine,
                             static_cast<cudaStream_t>(stream));
}

// Work items {q_start, q_len, q_pos0, blk_begin, blk_count, q_tile, kv_head,
// n_kv_tiles} (self-contained so the kernel never chases req_meta).  A query tile only needs the
// key tiles up to the slot holding its last query position (causal), so the
// count is found by a binary search over the table's logical block starts.
// Items are ordered for L2 reuse (see below).
int rcb_attn_plan(const int32_t* req_meta, int32_t n_req, const int32_t* blk_valid,
                  const int32_t* blk_pos, int32_t block_tokens, int32_t n_q_heads,
                  int32_t n_kv_heads, int32_t* work_out, int32_t cap, int32_t* n_work_out) {
  if (n_kv_heads <= 0 || n_q_heads % n_kv_heads != 0 || 128 % (n_q_heads / n_kv_heads) != 0)
    return rcb::set_error(RCB_ERR_ARG, "unsupported head grouping");
  const int g = n_q_heads / n_kv_heads;
  const int tq = 128 / g;  // tokens per 128-row query tile
  struct Item {
    int32_t r, qp, h, n0, n1;
    bool half0, half1;  // the tile's last KV tile needs only its first 64 key slots
  };
  const int kItemInts = 8;
  std::vector<Item> items;
  for (int32_t r = 0; r < n_req; ++r) {
    const int32_t q_len = req_meta[r * 5 + 1];
    const int32_t q_pos0 = req_meta[r * 5 + 2];
    const int32_t b0 = req_meta[r * 5 + 3];
    const int32_t nb = req_meta[r * 5 + 4];
    if (q_len <= 0) continue;
    if (nb <= 0) return rcb::set_error(RCB_ERR_ARG, "request with queries but no blocks");
    // KV tiles (128 key slots) query tile qt needs: up to the slot of its last token;
    // *half: that slot lies in the first 64 slots of the last tile
    auto tiles_of = [&](int32_t qt, bool* half) -> int32_t {
      *half = false;
      if (qt * tq >= q_len) return 0;
      const int32_t max_qp = q_pos0 + std::min(q_len, (qt + 1) * tq) - 1;
      int32_t lo = 0, hi = nb - 1;  // last block whose start <= max_qp
      while (lo < hi) {
        const int32_t mid = (lo + hi + 1) / 2;
        if (blk_pos[b0 + mid] <= max_qp) lo = mid;
        else hi = mid - 1;
      }
      const int32_t off = std::min(blk_valid[b0 + lo] - 1, max_qp - blk_pos[b0 + lo]);
      const int32_t slot = lo * block_tokens + std::max(0, off);
      *half = (slot % 128) < 64;
      return slot / 128 + 1;
    };
    const int32_t n_pairs = (q_len + 2 * tq - 1) / (2 * tq);
    for (int32_t qp = 0; qp < n_pairs; ++qp) {
      bool h0 = false, h1 = false;
      const int32_t n0 = tiles_of(2 * qp, &h0), n1 = tiles_of(2 * qp + 1, &h1);
      if (n0 > 0x7fff || n1 > 0x7fff) return rcb::set_error(RCB_ERR_ARG, "sequence too long");
      for (int32_t h = 0; h < n_kv_heads; ++h) items.push_back({r, qp, h, n0, n1, h0, h1});
    }
  }
  // L2 locality: the ~148 CTAs of a persistent launch take consecutive items,
  // so keep all q-tiles of one (request, kv head) adjacent — they re-read the
  // same K/V pages.  Requests go heaviest first, q-tiles longest first.
  std::vector<int64_t> req_work(n_req, 0);
  for (const Item& it : items) req_work[it.r] += it.n0 + it.n1;
  std::stable_sort(items.begin(), items.end(), [&](const Item& a, const Item& b) {
    if (a.r != b.r) {
      if (req_work[a.r] != req_work[b.r]) return req_work[a.r] > req_work[b.r];
      return a.r < b.r;
    }
    if (a.h != b.h) return a.h < b.h;
    return a.n0 + a.n1 > b.n0 + b.n1;
  });
  if (n_work_out) *n_work_out = static_cast<int32_t>(items.size());
  if (static_cast<int32_t>(items.size()) > cap)
    return rcb::set_error(RCB_ERR_ARG, "work capacity too small");
  for (size_t i = 0; i < items.size(); ++i) {
    const int32_t* m = req_meta + items[i].r * 5;
    int32_t* w = work_out + kItemInts * i;
    w[0] = m[0];  // q_start
    w[1] = m[1];  // q_len
    w[2] = m[2];  // q_pos0
    w[3] = m[3];  // blk_begin
    w[4] = m[4];  // blk_count
    w[5] = items[i].qp;
    w[6] = items[i].h;
    // n0 | half0 << 15 | n1 << 16 | half1 << 31
    const uint32_t packed = static_cast<uint32_t>(items[i].n0) |
                            (static_cast<uint32_t>(items[i].half0) << 15) |
                            (static_cast<uint32_t>(items[i].n1) << 16) |
                            (static_cast<uint32_t>(items[i].half1) << 31);
    w[7] = static_cast<int32_t>(packed);
  }
  return RCB_OK;
}

}  // extern "C"
