// rcb_internal.h — shared internals of libragcache_b200 (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/ragcache_b200.h"

namespace rcb {

// thread-local last-error text surfaced through rcb_last_error()
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda),
// bf16 elements, SWIZZLE_128B, OOB fill zero.  strides are in bytes for dims 1..rank-1.
int encode_tma_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                    const uint64_t* strides, const uint32_t* box);

int prefix_prefill(const void* q, int64_t q_row_stride, void* o, int total_q_tokens,
                   int n_q_heads, const void* kv_pool, int64_t num_pool_blocks, int block_tokens,
                   int n_layers, int n_kv_heads, int head_dim, int layer, const int* req_meta,
                   const int* blk_ids, const int* blk_valid, const int* blk_pos, const int* work,
                   int n_work, float softmax_scale, const void* rope_table, int work_flags,
                   void* part_ws, int n_part_slots, const int* combine, int n_combine,
                   cudaStream_t stream);

// block copy with the (src, dst) block-index list passed by value in the launch
constexpr int kPairsPerLaunch = 1024;
struct BlockPairs {
  int32_t src[kPairsPerLaunch];
  int32_t dst[kPairsPerLaunch];
};
cudaError_t launch_block_copy_params(const void* src_base, void* dst_base, int64_t block_bytes,
                                     const BlockPairs& pairs, int n, cudaStream_t stream);
cudaError_t launch_block_copy_dev(const void* src_base, void* dst_base, int64_t block_bytes,
                                  const int32_t* pairs_dev, int n, cudaStream_t stream);

}  // namespace rcb
