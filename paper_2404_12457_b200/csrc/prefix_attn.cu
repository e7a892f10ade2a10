// prefix_attn.cu — prefix-aware prefill attention over the paged doc-KV pool.
//
// Replaces the reference's latency stand-in T(alpha, beta)
// (ragsim cost_model.py:106-117 `interpolate`, called at simulator.py:506 and
// tree.py:240): here the alpha cached tokens are READ from knowledge-tree node
// blocks through a block table, and only the beta suffix tokens (miss docs +
// prompt) are computed as queries.
//
// One CTA = one work item (request, query tile, kv head):
//   * 128 query rows = (128/G tokens) x (G query heads sharing the kv head)
//   * K/V tiles of 128 key slots = 128/BT pool blocks, TMA-loaded (SW128)
//   * S = Q K^T and O += P V on tcgen05 (fp32 accumulators in TMEM)
//   * online softmax in registers, one thread per row (warps 0-3),
//     lazily rescaled O (only when the running max grows by > 2^8)
// Warp roles: 0-3 softmax/epilogue, 4 TMA producer, 5 MMA issuer + TMEM owner.
//
// Key slots carry holes (node tails: a block holds `valid` <= BT tokens), so
// each block also carries its logical start position; a slot is attended iff
// off < valid && pos <= query_pos (causal on logical positions).
#include "sm100.cuh"
#include "rcb_internal.h"

namespace rcb {

namespace attn {

constexpr int kThreads = 192;
constexpr int kRows = 128;
constexpr int kKeys = 128;  // key slots per KV tile
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int HD>
struct Smem {
  static constexpr uint32_t kHalves = HD / 64;
  static constexpr uint32_t kQ = kHalves * 16384;
  static constexpr uint32_t kKV = kHalves * 16384;  // one K or V stage
  static constexpr uint32_t kP = 2 * 16384;
  static constexpr uint32_t offQ = 0;
  static constexpr uint32_t offK = offQ + kQ;
  static constexpr uint32_t offV = offK + 2 * kKV;
  static constexpr uint32_t offP = offV + 2 * kKV;
  static constexpr uint32_t offBar = offP + kP;
  static constexpr uint32_t kTotal = offBar + 256 + 1024;  // + alignment slack
};

enum Bar {
  kQFull = 0,
  kKFull0 = 1,
  kVFull0 = 3,
  kKVEmpty0 = 5,
  kSFull0 = 7,
  kSFree0 = 9,
  kPFull = 11,
  kPFree = 12,
  kOFull = 13,
  kNumBars = 14
};

template <int HD, int G, int BT>
__global__ void __launch_bounds__(kThreads, 1)
    prefix_prefill_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_kv,
                          __nv_bfloat16* __restrict__ out, int n_q_heads, int layer,
                          const int* __restrict__ req_meta, const int* __restrict__ blk_ids,
                          const int* __restrict__ blk_valid, const int* __restrict__ blk_pos,
                          const int* __restrict__ work, float scale_log2) {
  using S = Smem<HD>;
  constexpr int TQ = kRows / G;
  constexpr int BPT = kKeys / BT;  // pool blocks per KV tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + S::offQ;
  uint8_t* sK = smem + S::offK;
  uint8_t* sV = smem + S::offV;
  uint8_t* sP = smem + S::offP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::offBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + kNumBars);

  const int warp = threadIdx.x >> 5;
  const int item = blockIdx.x;
  const int req = work[item * 4 + 0];
  const int qt = work[item * 4 + 1];
  const int kvh = work[item * 4 + 2];
  const int n_tiles = work[item * 4 + 3];
  const int q_start = req_meta[req * 5 + 0];
  const int q_len = req_meta[req * 5 + 1];
  const int q_pos0 = req_meta[req * 5 + 2];
  const int blk_begin = req_meta[req * 5 + 3];
  const int blk_count = req_meta[req * 5 + 4];

  if (threadIdx.x == 0) {
    mbar_init(&bar[kQFull], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar[kKFull0 + s], 1);
      mbar_init(&bar[kVFull0 + s], 1);
      mbar_init(&bar[kKVEmpty0 + s], 1);
      mbar_init(&bar[kSFull0 + s], 1);
      mbar_init(&bar[kSFree0 + s], kRows);
    }
    mbar_init(&bar[kPFull], kRows);
    mbar_init(&bar[kPFree], 1);
    mbar_init(&bar[kOFull], 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_kv);
      mbar_arrive_expect_tx(&bar[kQFull], S::kQ);
      for (int h = 0; h < (int)S::kHalves; ++h)
        tma_load_3d(sQ + h * 16384, &tm_q, &bar[kQFull], h * 64, kvh * G, q_start + qt * TQ);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        mbar_wait(&bar[kKVEmpty0 + st], ((j >> 1) & 1) ^ 1);
        int ids[BPT];
#pragma unroll
        for (int b = 0; b < BPT; ++b) {
          const int sb = j * BPT + b;
          // slots past the table load a real (finite) block; they are masked
          ids[b] = blk_ids[blk_begin + (sb < blk_count ? sb : 0)];
        }
        mbar_arrive_expect_tx(&bar[kKFull0 + st], S::kKV);
#pragma unroll
        for (int b = 0; b < BPT; ++b)
          for (int h = 0; h < (int)S::kHalves; ++h)
            tma_load_5d(sK + st * S::kKV + h * 16384 + b * BT * 128, &tm_kv, &bar[kKFull0 + st],
                        h * 64, 0, kvh, 2 * layer, ids[b]);
        mbar_arrive_expect_tx(&bar[kVFull0 + st], S::kKV);
#pragma unroll
        for (int b = 0; b < BPT; ++b)
          for (int h = 0; h < (int)S::kHalves; ++h)
            tma_load_5d(sV + st * S::kKV + h * 16384 + b * BT * 128, &tm_kv, &bar[kVFull0 + st],
                        h * 64, 0, kvh, 2 * layer + 1, ids[b]);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, kKeys, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, HD, 0, 1);
      const uint32_t q_base = smem_u32(sQ);
      const uint32_t k_base = smem_u32(sK);
      const uint32_t v_base = smem_u32(sV);
      const uint32_t p_base = smem_u32(sP);
      mbar_wait(&bar[kQFull], 0);
      tc_fence_after();
      auto issue_qk = [&](int j) {
        const int st = j & 1;
        mbar_wait(&bar[kKFull0 + st], (j >> 1) & 1);
        mbar_wait(&bar[kSFree0 + st], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + st * kKeys;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint64_t a = sw128_desc(q_base + off, 16, 1024);
          const uint64_t b = sw128_desc(k_base + st * S::kKV + off, 16, 1024);
          umma_bf16_ss(d, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&bar[kSFull0 + st]);
      };
      issue_qk(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) issue_qk(j + 1);
        const int st = j & 1;
        mbar_wait(&bar[kPFull], j & 1);
        mbar_wait(&bar[kVFull0 + st], (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kKeys / 16; ++kk) {
          const uint64_t a = sw128_desc(p_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          // V tile is [half][128 keys][64]: MN-major, halves 16 KB apart (LBO)
          const uint64_t b = sw128_desc(v_base + st * S::kKV + kk * 2048, 16384, 1024);
          umma_bf16_ss(tmem + 256, a, b, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&bar[kKVEmpty0 + st]);
        umma_commit(&bar[kPFree]);
      }
      umma_commit(&bar[kOFull]);
    }
  } else {
    // ------------------------------------------------------------ softmax rows
    const int row = threadIdx.x;  // == TMEM lane
    const int t_local = row / G;
    const int h_local = row % G;
    const int tok = qt * TQ + t_local;
    const bool row_valid = tok < q_len;
    const int qp = q_pos0 + tok;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    float m = -INFINITY;  // running max (scaled, log2 domain); may be stale by < 2^8
    float l = 0.f;
    float s[kKeys];
    for (int j = 0; j < n_tiles; ++j) {
      // tile metadata (broadcast loads)
      int vv[BPT], pp[BPT];
      bool all_valid = true;
      int max_pos = -1;
#pragma unroll
      for (int b = 0; b < BPT; ++b) {
        const int sb = j * BPT + b;
        const bool in = sb < blk_count;
        vv[b] = in ? blk_valid[blk_begin + sb] : 0;
        pp[b] = in ? blk_pos[blk_begin + sb] : 0;
        all_valid &= (vv[b] == BT);
        max_pos = max(max_pos, pp[b] + vv[b] - 1);
      }
      const int st = j & 1;
      mbar_wait(&bar[kSFull0 + st], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < kKeys / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(t_row + st * kKeys + c * 32, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(r[i]);
      }
      tc_fence_before();
      mbar_arrive(&bar[kSFree0 + st]);

      if (!all_valid || max_pos > qp) {
#pragma unroll
        for (int c = 0; c < kKeys; ++c) {
          const int b = c / BT, off = c % BT;
          const bool ok = off < vv[b] && pp[b] + off <= qp;
          s[c] = ok ? s[c] : -INFINITY;
        }
      }
      float tmax = -INFINITY;
#pragma unroll
      for (int c = 0; c < kKeys; ++c) tmax = fmaxf(tmax, s[c]);
      tmax *= scale_log2;
      float alpha = 1.f;
      bool rescale = false;
      if (j == 0) {
        m = (tmax == -INFINITY) ? 0.f : tmax;
      } else if (tmax > m + kRescaleThreshold) {
        alpha = exp2f(m - tmax);
        m = tmax;
        l *= alpha;
        rescale = true;
      }
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < kKeys; ++c) {
        const float p = exp2f(fmaf(s[c], scale_log2, -m));
        s[c] = p;
        rs += p;
      }
      l += rs;
      if (j > 0) {
        mbar_wait(&bar[kPFree], (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(t_row + 256 + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st32(t_row + 256 + c * 32, r);
          }
          tmem_wait_st();
        }
      }
      // P row -> smem, K-major SW128 (two 64-key regions)
      uint8_t* prow = sP + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
      for (int cc = 0; cc < kKeys / 8; ++cc) {
        uint4 v;
        v.x = pack_bf16(s[cc * 8 + 0], s[cc * 8 + 1]);
        v.y = pack_bf16(s[cc * 8 + 2], s[cc * 8 + 3]);
        v.z = pack_bf16(s[cc * 8 + 4], s[cc * 8 + 5]);
        v.w = pack_bf16(s[cc * 8 + 6], s[cc * 8 + 7]);
        *reinterpret_cast<uint4*>(prow + (cc >> 3) * 16384 + (((cc & 7) ^ (row & 7)) << 4)) = v;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bar[kPFull]);
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(&bar[kOFull], 0);
    tc_fence_after();
    const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
    __nv_bfloat16* orow =
        out + (static_cast<int64_t>(q_start + tok) * n_q_heads + kvh * G + h_local) * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(t_row + 256 + c * 32, r);
      tmem_wait_ld();
      if (row_valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 v;
          v.x = pack_bf16(__uint_as_float(r[i + 0]) * inv_l, __uint_as_float(r[i + 1]) * inv_l);
          v.y = pack_bf16(__uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
          v.z = pack_bf16(__uint_as_float(r[i + 4]) * inv_l, __uint_as_float(r[i + 5]) * inv_l);
          v.w = pack_bf16(__uint_as_float(r[i + 6]) * inv_l, __uint_as_float(r[i + 7]) * inv_l);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = v;
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int HD, int G, int BT>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tkv, void* out, int n_q_heads,
                     int layer, const int* req_meta, const int* blk_ids, const int* blk_valid,
                     const int* blk_pos, const int* work, int n_work, float scale_log2,
                     cudaStream_t stream) {
  auto kern = prefix_prefill_kernel<HD, G, BT>;
  const uint32_t smem = Smem<HD>::kTotal;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<n_work, kThreads, smem, stream>>>(tq, tkv, static_cast<__nv_bfloat16*>(out), n_q_heads,
                                          layer, req_meta, blk_ids, blk_valid, blk_pos, work,
                                          scale_log2);
  return cudaGetLastError();
}

template <int HD, int G>
cudaError_t launch_bt(int bt, const CUtensorMap& tq, const CUtensorMap& tkv, void* out,
                      int n_q_heads, int layer, const int* rm, const int* bi, const int* bv,
                      const int* bp, const int* work, int n_work, float sl2, cudaStream_t st) {
  switch (bt) {
    case 16: return launch_t<HD, G, 16>(tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, st);
    case 32: return launch_t<HD, G, 32>(tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, st);
    case 64: return launch_t<HD, G, 64>(tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, st);
    case 128: return launch_t<HD, G, 128>(tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int HD>
cudaError_t launch_g(int g, int bt, const CUtensorMap& tq, const CUtensorMap& tkv, void* out,
                     int n_q_heads, int layer, const int* rm, const int* bi, const int* bv,
                     const int* bp, const int* work, int n_work, float sl2, cudaStream_t st) {
  switch (g) {
    case 1: return launch_bt<HD, 1>(bt, tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, st);
    case 2: return launch_bt<HD, 2>(bt, tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, st);
    case 4: return launch_bt<HD, 4>(bt, tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, st);
    case 8: return launch_bt<HD, 8>(bt, tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace attn

int prefix_prefill(const void* q, void* o, int total_q_tokens, int n_q_heads, const void* kv_pool,
                   int64_t num_pool_blocks, int block_tokens, int n_layers, int n_kv_heads,
                   int head_dim, int layer, const int* req_meta, const int* blk_ids,
                   const int* blk_valid, const int* blk_pos, const int* work, int n_work,
                   float softmax_scale, cudaStream_t stream) {
  if (n_work == 0) return RCB_OK;
  if (head_dim != 64 && head_dim != 128) return set_error(RCB_ERR_ARG, "head_dim must be 64 or 128");
  if (n_kv_heads <= 0 || n_q_heads % n_kv_heads != 0) return set_error(RCB_ERR_ARG, "bad head counts");
  const int g = n_q_heads / n_kv_heads;
  if (layer < 0 || layer >= n_layers) return set_error(RCB_ERR_ARG, "layer out of range");
  CUtensorMap tq, tkv;
  {
    const uint64_t dims[3] = {(uint64_t)head_dim, (uint64_t)n_q_heads, (uint64_t)total_q_tokens};
    const uint64_t strides[2] = {(uint64_t)head_dim * 2, (uint64_t)n_q_heads * head_dim * 2};
    const uint32_t box[3] = {64, (uint32_t)g, (uint32_t)(128 / g)};
    int rc = encode_tma_bf16(&tq, q, 3, dims, strides, box);
    if (rc != RCB_OK) return rc;
  }
  {
    const uint64_t blk_bytes =
        (uint64_t)n_layers * 2 * n_kv_heads * block_tokens * head_dim * 2;
    const uint64_t dims[5] = {(uint64_t)head_dim, (uint64_t)block_tokens, (uint64_t)n_kv_heads,
                              (uint64_t)(2 * n_layers), (uint64_t)num_pool_blocks};
    const uint64_t strides[4] = {(uint64_t)head_dim * 2, (uint64_t)block_tokens * head_dim * 2,
                                 (uint64_t)n_kv_heads * block_tokens * head_dim * 2, blk_bytes};
    const uint32_t box[5] = {64, (uint32_t)block_tokens, 1, 1, 1};
    int rc = encode_tma_bf16(&tkv, kv_pool, 5, dims, strides, box);
    if (rc != RCB_OK) return rc;
  }
  const float sl2 = softmax_scale * 1.4426950408889634f;
  cudaError_t e =
      head_dim == 128
          ? attn::launch_g<128>(g, block_tokens, tq, tkv, o, n_q_heads, layer, req_meta, blk_ids,
                                blk_valid, blk_pos, work, n_work, sl2, stream)
          : attn::launch_g<64>(g, block_tokens, tq, tkv, o, n_q_heads, layer, req_meta, blk_ids,
                               blk_valid, blk_pos, work, n_work, sl2, stream);
  if (e != cudaSuccess) return set_cuda_error(e, "prefix_prefill launch");
  return RCB_OK;
}

}  // namespace rcb
