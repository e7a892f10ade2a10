// kv_ops.cu — KV block movement and paged KV writes.
//
// (1) block gather/scatter: the data path behind the knowledge tree's tier
//     transitions (swap-out tree.py:460-473, swap-in tree.py:296-318) which the
//     reference only prices with transfer_time (cost_model.py:120-124).  One
//     HBM->HBM copies (staging gather/scatter, compaction) run on the TMA engine
//     (cp.async.bulk through an smem ring, one issuing lane per CTA); HBM<->mapped
//     pinned host (zero-copy swap) uses 16-byte vector accesses, 8 loads in flight
//     per thread; both grid-stride over (pair, 32 KB chunk) units.
// (2) RoPE + paged KV write: the suffix tokens' K/V (miss docs + prompt) are
//     rotated and scattered straight into their reserved pool blocks, so a
//     committed node adopts them with no copy (tree.py:252-294 insert_path).
#include <algorithm>
#include <cuda_bf16.h>

#include "rcb_internal.h"
#include "sm100.cuh"

#ifndef RCB_PDL
#define RCB_PDL 1
#endif

namespace rcb {

namespace {

constexpr int kCopyThreads = 256;
constexpr int kCopyUnroll = 8;
constexpr int64_t kChunk = int64_t(kCopyThreads) * 16 * kCopyUnroll;  // 32 KB

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void copy_unit(const uint8_t* __restrict__ src,
                                          uint8_t* __restrict__ dst, int64_t block_bytes,
                                          int64_t chunk) {
  const int64_t base = chunk * kChunk + int64_t(threadIdx.x) * 16;
  uint4 v[kCopyUnroll];
  if (base + (kCopyUnroll - 1) * kCopyThreads * 16 + 16 <= block_bytes) {
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u)
      v[u] = ld_stream(reinterpret_cast<const uint4*>(src + base + u * kCopyThreads * 16));
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u)
      *reinterpret_cast<uint4*>(dst + base + u * kCopyThreads * 16) = v[u];
  } else {
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) {
      const int64_t off = base + u * kCopyThreads * 16;
      if (off + 16 <= block_bytes) v[u] = ld_stream(reinterpret_cast<const uint4*>(src + off));
    }
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) {
      const int64_t off = base + u * kCopyThreads * 16;
      if (off + 16 <= block_bytes) *reinterpret_cast<uint4*>(dst + off) = v[u];
    }
  }
}

__global__ void __launch_bounds__(kCopyThreads)
    block_copy_params_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                             int64_t block_bytes, const __grid_constant__ BlockPairs pairs, int n) {
  const int64_t cpb = (block_bytes + kChunk - 1) / kChunk;
  const int64_t units = cpb * n;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int i = static_cast<int>(u / cpb);
    const int64_t c = u - i * cpb;
    copy_unit(src + int64_t(pairs.src[i]) * block_bytes, dst + int64_t(pairs.dst[i]) * block_bytes,
              block_bytes, c);
  }
}

__global__ void __launch_bounds__(kCopyThreads)
    block_copy_dev_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                          int64_t block_bytes, const int32_t* __restrict__ pairs, int n) {
  const int64_t cpb = (block_bytes + kChunk - 1) / kChunk;
  const int64_t units = cpb * n;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int i = static_cast<int>(u / cpb);
    const int64_t c = u - i * cpb;
    copy_unit(src + int64_t(pairs[2 * i]) * block_bytes,
              dst + int64_t(pairs[2 * i + 1]) * block_bytes, block_bytes, c);
  }
}

// ---------------------------------------------------------------- TMA bulk copy
// HBM -> HBM block copy on the TMA engine: one elected lane per CTA streams its
// (pair, 32 KB chunk) units through a kBulkStages-deep smem ring with
// cp.async.bulk (global -> smem, mbarrier complete_tx) and cp.async.bulk
// (smem -> global, bulk group).  No data passes through registers; the CTA is one
// warp.  Device memory on both sides (the zero-copy host path keeps the SIMT kernel).
constexpr int kBulkChunk = 32768;
constexpr int kBulkStages = 4;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}

template <bool kByValue>
__global__ void __launch_bounds__(32)
    block_copy_bulk_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                           int64_t block_bytes, const __grid_constant__ BlockPairs pairs,
                           const int32_t* __restrict__ pairs_dev, int n) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kBulkStages];
  if (!elect_one()) return;
  const int64_t cpb = (block_bytes + kBulkChunk - 1) / kBulkChunk;
  const int64_t units = cpb * n;
  // this CTA's units: u_k = blockIdx.x + k * gridDim.x
  const int64_t mine = units > blockIdx.x ? (units - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  for (int s = 0; s < kBulkStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto unit = [&](int64_t k, const uint8_t*& s, uint8_t*& d, uint32_t& bytes) {
    const int64_t u = blockIdx.x + k * gridDim.x;
    const int i = static_cast<int>(u / cpb);
    const int64_t c = u - i * cpb;
    const int32_t ps = kByValue ? pairs.src[i] : pairs_dev[2 * i];
    const int32_t pd = kByValue ? pairs.dst[i] : pairs_dev[2 * i + 1];
    const int64_t off = c * kBulkChunk;
    s = src + int64_t(ps) * block_bytes + off;
    d = dst + int64_t(pd) * block_bytes + off;
    const int64_t rem = block_bytes - off;
    bytes = static_cast<uint32_t>(rem < kBulkChunk ? rem : kBulkChunk);
  };
  auto load = [&](int64_t k) {
    const uint8_t* s;
    uint8_t* d;
    uint32_t bytes;
    unit(k, s, d, bytes);
    const int st = static_cast<int>(k % kBulkStages);
    const uint32_t bar = smem_u32(&full[st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    bulk_g2s(smem_u32(ring + st * kBulkChunk), s, bytes, bar);
  };
  for (int64_t k = 0; k < mine && k < kBulkStages; ++k) load(k);
  for (int64_t k = 0; k < mine; ++k) {
    const int st = static_cast<int>(k % kBulkStages);
    const uint32_t bar = smem_u32(&full[st]);
    const uint32_t ph = static_cast<uint32_t>((k / kBulkStages) & 1);
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra W_%=;\n\t}" ::"r"(bar), "r"(ph)
        : "memory");
    const uint8_t* s;
    uint8_t* d;
    uint32_t bytes;
    unit(k, s, d, bytes);
    bulk_s2g(d, smem_u32(ring + st * kBulkChunk), bytes);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill the stage the previous store read from (at most the newest store pending)
    if (k >= 1 && k - 1 + kBulkStages < mine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(k - 1 + kBulkStages);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int copy_grid(int64_t block_bytes, int n) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t units = ((block_bytes + kChunk - 1) / kChunk) * n;
  const int64_t cap = int64_t(sms) * 4;
  return static_cast<int>(units < cap ? units : cap);
}

// ------------------------------------------------------------------ RoPE + write
// One CTA per token.  cos/sin of the token's head_dim/2 frequencies are
// computed once into shared memory and shared by every q/k head; each thread
// then rotates 8-element (16 B) chunks of x[i] and x[i + d/2] and copies V
// chunks straight into the token's pool slot.
constexpr int kRopeThreads = 128;

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

__global__ void __launch_bounds__(kRopeThreads)
    kv_write_rope_kernel(const __nv_bfloat16* __restrict__ q, int64_t q_stride,
                         const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
                         int64_t kv_stride, __nv_bfloat16* __restrict__ q_out,
                         const int32_t* __restrict__ positions, const int32_t* __restrict__ slots,
                         int n_q_heads, __nv_bfloat16* __restrict__ pool, int block_tokens,
                         int64_t block_elems, int n_kv_heads, int head_dim, int layer,
                         float log2_theta) {
  __shared__ float s_cos[128], s_sin[128];
  const int t = blockIdx.x;
  const int half = head_dim / 2;
  const float pos = static_cast<float>(positions[t]);
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float inv_freq = exp2f(-(2.f * i / head_dim) * log2_theta);
    sincosf(pos * inv_freq, &s_sin[i], &s_cos[i]);
  }
  const int slot = slots[t];
  const int blk = slot / block_tokens;
  const int off = slot - blk * block_tokens;
  const int64_t tile = int64_t(block_tokens) * head_dim;
  __nv_bfloat16* kbase = pool + int64_t(blk) * block_elems +
                         int64_t(2 * layer) * n_kv_heads * tile + int64_t(off) * head_dim;
  __nv_bfloat16* vbase = kbase + int64_t(n_kv_heads) * tile;
  __syncthreads();
  const int cph = half / 8;  // 16-byte chunks per half row
  // q == nullptr: K/V only (Q's RoPE is fused into the attention kernel)
  const int q_heads = q != nullptr ? n_q_heads : 0;
  const int rot_units = (q_heads + n_kv_heads) * cph;
  const int v_units = n_kv_heads * (head_dim / 8);
  for (int u = threadIdx.x; u < rot_units + v_units; u += blockDim.x) {
    if (u < rot_units) {
      const int h = u / cph;
      const int c = (u - h * cph) * 8;
      const __nv_bfloat16* src;
      __nv_bfloat16* dst;
      if (h < q_heads) {
        src = q + int64_t(t) * q_stride + int64_t(h) * head_dim;
        dst = q_out + (int64_t(t) * n_q_heads + h) * head_dim;
      } else {
        src = k + int64_t(t) * kv_stride + int64_t(h - q_heads) * head_dim;
        dst = kbase + int64_t(h - q_heads) * tile;
      }
      float x0[8], x1[8], y0[8], y1[8];
      unpack8(*reinterpret_cast<const uint4*>(src + c), x0);
      unpack8(*reinterpret_cast<const uint4*>(src + c + half), x1);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float cs = s_cos[c + e], sn = s_sin[c + e];
        y0[e] = x0[e] * cs - x1[e] * sn;
        y1[e] = x1[e] * cs + x0[e] * sn;
      }
      *reinterpret_cast<uint4*>(dst + c) = pack8(y0);
      *reinterpret_cast<uint4*>(dst + c + half) = pack8(y1);
    } else {
      const int j = u - rot_units;
      const int h = j / (head_dim / 8);
      const int c = (j - h * (head_dim / 8)) * 8;
      *reinterpret_cast<uint4*>(vbase + int64_t(h) * tile + c) =
          *reinterpret_cast<const uint4*>(v + int64_t(t) * kv_stride + int64_t(h) * head_dim + c);
    }
  }
}

// Table-driven variant: cos/sin come from the rcb_rope_table (the same table the attention
// kernel rotates Q with, computed with the same formula), so no per-token sincosf and no
// __syncthreads; kKvTok tokens per CTA, consecutive threads take consecutive 16 B chunks
// of a token's heads (coalesced reads of the QKV row, 256 B runs into each pool slot).
#ifndef RCB_KV_TOK
#define RCB_KV_TOK 8
#endif
#ifndef RCB_KV_UNROLL
#define RCB_KV_UNROLL 1
#endif
constexpr int kKvTok = RCB_KV_TOK;
constexpr int kKvUnroll = RCB_KV_UNROLL;
constexpr int kKvTabThreads = 256;
#ifndef RCB_KV_UNITS
#define RCB_KV_UNITS 1024
#endif
constexpr int kKvTabUnits = RCB_KV_UNITS;  // chunk units per CTA the token count aims at
#ifndef RCB_KV_V32
#define RCB_KV_V32 1
#endif
constexpr bool kKvV32 = RCB_KV_V32 != 0;

__global__ void __launch_bounds__(kKvTabThreads)
    kv_write_rope_tab_kernel(const __nv_bfloat16* __restrict__ q, int64_t q_stride,
                             const __nv_bfloat16* __restrict__ k,
                             const __nv_bfloat16* __restrict__ v, int64_t kv_stride,
                             __nv_bfloat16* __restrict__ q_out,
                             const int32_t* __restrict__ positions,
                             const int32_t* __restrict__ slots, int n_tokens, int n_q_heads,
                             __nv_bfloat16* __restrict__ pool, int block_tokens,
                             int64_t block_elems, int n_kv_heads, int head_dim, int layer,
                             const float4* __restrict__ table, int tok_per_cta) {
#if RCB_PDL
  // programmatic dependent launch: the attention launch that follows may start its
  // prologue on SMs this grid frees (it waits for our writes before reading K/V)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  const int half = head_dim / 2;
  const int cph = half / 8;  // 16-byte chunks per half row
  const int q_heads = q != nullptr ? n_q_heads : 0;
  const int rot_units = (q_heads + n_kv_heads) * cph;
  // V moves in 32-byte chunks when rows allow (half the memory instructions of 16-byte ones)
  const int vw = (kKvV32 && kv_stride % 16 == 0 && head_dim % 16 == 0 &&
                  (reinterpret_cast<uintptr_t>(v) & 31) == 0 &&
                  (reinterpret_cast<uintptr_t>(pool) & 31) == 0) ? 16 : 8;
  const int per_tok = rot_units + n_kv_heads * (head_dim / vw);
  const int t0 = blockIdx.x * tok_per_cta;
  const int n = min(tok_per_cta, n_tokens - t0) * per_tok;
  const int64_t tile = int64_t(block_tokens) * head_dim;
#pragma unroll kKvUnroll
  for (int u = threadIdx.x; u < n; u += kKvTabThreads) {
    const int tt = u / per_tok;
    const int j = u - tt * per_tok;
    const int t = t0 + tt;
    const int slot = __ldg(slots + t);
    const int blk = slot / block_tokens;
    const int off = slot - blk * block_tokens;
    __nv_bfloat16* kbase = pool + int64_t(blk) * block_elems +
                           int64_t(2 * layer) * n_kv_heads * tile + int64_t(off) * head_dim;
    if (j < rot_units) {
      const int h = j / cph;
      const int c = (j - h * cph) * 8;
      const __nv_bfloat16* src;
      __nv_bfloat16* dst;
      if (h < q_heads) {
        src = q + int64_t(t) * q_stride + int64_t(h) * head_dim;
        dst = q_out + (int64_t(t) * n_q_heads + h) * head_dim;
      } else {
        src = k + int64_t(t) * kv_stride + int64_t(h - q_heads) * head_dim;
        dst = kbase + int64_t(h - q_heads) * tile;
      }
      const uint4 a = *reinterpret_cast<const uint4*>(src + c);
      const uint4 b = *reinterpret_cast<const uint4*>(src + c + half);
      // table row of this position: (cos, sin) of frequencies c .. c+7 = 4 float4
      const float4* tab = table + (int64_t(__ldg(positions + t)) * half + c) / 2;
      float cs[8], sn[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 f = __ldg(tab + e);
        cs[2 * e] = f.x;
        sn[2 * e] = f.y;
        cs[2 * e + 1] = f.z;
        sn[2 * e + 1] = f.w;
      }
      float x0[8], x1[8], y0[8], y1[8];
      unpack8(a, x0);
      unpack8(b, x1);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        y0[e] = x0[e] * cs[e] - x1[e] * sn[e];
        y1[e] = x1[e] * cs[e] + x0[e] * sn[e];
      }
      *reinterpret_cast<uint4*>(dst + c) = pack8(y0);
      *reinterpret_cast<uint4*>(dst + c + half) = pack8(y1);
    } else {
      const int jj = j - rot_units;
      const int h = jj / (head_dim / vw);
      const int c = (jj - h * (head_dim / vw)) * vw;
      const __nv_bfloat16* vs = v + int64_t(t) * kv_stride + int64_t(h) * head_dim + c;
      __nv_bfloat16* vd = kbase + int64_t(n_kv_heads + h) * tile + c;
      if (vw == 16) {
        uint4 lo, hi;
        asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y),
                       "=r"(hi.z), "=r"(hi.w)
                     : "l"(vs));
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(vd),
                     "r"(lo.x), "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z),
                     "r"(hi.w)
                     : "memory");
      } else {
        *reinterpret_cast<uint4*>(vd) = *reinterpret_cast<const uint4*>(vs);
      }
    }
  }
}

}  // namespace

#ifndef RCB_BULK_COPY
#define RCB_BULK_COPY 1
#endif

namespace {
// both bases in device memory (not mapped host): the TMA bulk path applies
bool both_device(const void* a, const void* b) {
  if (!RCB_BULK_COPY) return false;
  for (const void* p : {a, b}) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeDevice) return false;
  }
  return true;
}

template <bool kByValue>
cudaError_t launch_bulk(const void* src_base, void* dst_base, int64_t block_bytes,
                        const BlockPairs* pairs, const int32_t* pairs_dev, int n,
                        cudaStream_t stream) {
  static bool attr = false;
  constexpr int smem = kBulkStages * kBulkChunk;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(block_copy_bulk_kernel<kByValue>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t units = ((block_bytes + kBulkChunk - 1) / kBulkChunk) * n;
  const int grid = static_cast<int>(units < sms ? units : sms);  // one CTA per SM (smem)
  static const BlockPairs kNone{};
  block_copy_bulk_kernel<kByValue><<<grid, 32, smem, stream>>>(
      static_cast<const uint8_t*>(src_base), static_cast<uint8_t*>(dst_base), block_bytes,
      pairs ? *pairs : kNone, pairs_dev, n);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_block_copy_params(const void* src_base, void* dst_base, int64_t block_bytes,
                                     const BlockPairs& pairs, int n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (both_device(src_base, dst_base))
    return launch_bulk<true>(src_base, dst_base, block_bytes, &pairs, nullptr, n, stream);
  block_copy_params_kernel<<<copy_grid(block_bytes, n), kCopyThreads, 0, stream>>>(
      static_cast<const uint8_t*>(src_base), static_cast<uint8_t*>(dst_base), block_bytes, pairs,
      n);
  return cudaGetLastError();
}

cudaError_t launch_block_copy_dev(const void* src_base, void* dst_base, int64_t block_bytes,
                                  const int32_t* pairs_dev, int n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (both_device(src_base, dst_base))
    return launch_bulk<false>(src_base, dst_base, block_bytes, nullptr, pairs_dev, n, stream);
  block_copy_dev_kernel<<<copy_grid(block_bytes, n), kCopyThreads, 0, stream>>>(
      static_cast<const uint8_t*>(src_base), static_cast<uint8_t*>(dst_base), block_bytes,
      pairs_dev, n);
  return cudaGetLastError();
}

}  // namespace rcb

extern "C" int rcb_kv_block_copy(const void* src_base, void* dst_base, int64_t block_bytes,
                                 const int32_t* pairs_dev, int32_t n_pairs, void* stream) {
  if (block_bytes <= 0 || block_bytes % 16 != 0)
    return rcb::set_error(RCB_ERR_ARG, "block_bytes must be a positive multiple of 16");
  if (n_pairs < 0) return rcb::set_error(RCB_ERR_ARG, "negative pair count");
  cudaError_t e = rcb::launch_block_copy_dev(src_base, dst_base, block_bytes, pairs_dev, n_pairs,
                                             static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return rcb::set_cuda_error(e, "rcb_kv_block_copy");
  return RCB_OK;
}

namespace rcb {
namespace {
__global__ void rope_table_kernel(float2* __restrict__ out, int max_pos, int half, int head_dim,
                                  float log2_theta) {
  const int64_t n = int64_t(max_pos) * half;
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < n;
       u += int64_t(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(u / half);
    const int i = static_cast<int>(u - int64_t(p) * half);
    const float inv_freq = exp2f(-(2.f * i / head_dim) * log2_theta);
    float sn, cs;
    sincosf(static_cast<float>(p) * inv_freq, &sn, &cs);
    out[u] = make_float2(cs, sn);
  }
}
}  // namespace
}  // namespace rcb

extern "C" int rcb_rope_table(void* table_dev, int32_t max_pos, int32_t head_dim, float rope_theta,
                              void* stream) {
  if (max_pos <= 0 || head_dim <= 0 || head_dim % 2 != 0)
    return rcb::set_error(RCB_ERR_ARG, "bad rope table shape");
  const int half = head_dim / 2;
  const int64_t n = int64_t(max_pos) * half;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  rcb::rope_table_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<float2*>(table_dev), max_pos, half, head_dim, log2f(rope_theta));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rcb::set_cuda_error(e, "rcb_rope_table");
  return RCB_OK;
}

extern "C" int rcb_kv_write_rope_table(const void* q, int64_t q_stride, const void* k,
                                       const void* v, int64_t kv_stride, void* q_out,
                                       const int32_t* positions_dev, const int32_t* slots_dev,
                                       int32_t n_tokens, int32_t n_q_heads, void* kv_pool,
                                       int32_t block_tokens, int32_t n_layers,
                                       int32_t n_kv_heads, int32_t head_dim, int32_t layer,
                                       const void* rope_table_dev, void* stream) {
  if (n_tokens == 0) return RCB_OK;
  if (head_dim % 16 != 0 || head_dim > 256 || layer < 0 || layer >= n_layers)
    return rcb::set_error(RCB_ERR_ARG, "head_dim must be a multiple of 16 (<= 256), layer in range");
  if (q_stride % 8 != 0 || kv_stride % 8 != 0)
    return rcb::set_error(RCB_ERR_ARG, "q/kv row strides must be multiples of 8 elements");
  if (rope_table_dev == nullptr) return rcb::set_error(RCB_ERR_ARG, "rope table required");
  const int64_t block_elems = int64_t(n_layers) * 2 * n_kv_heads * block_tokens * head_dim;
  // tokens per CTA: kKvTok at GQA widths (Mistral-7B: 128 chunk units per token, 4 per
  // thread); wide MHA rows (LLaMA2: 512-640 units per token) take fewer tokens per CTA so
  // each thread keeps ~4 units and the grid spans more waves
  const int per_tok = ((q != nullptr ? n_q_heads : 0) + 2 * n_kv_heads) * (head_dim / 16);
  const int tpc = std::max(1, std::min(rcb::kKvTok, rcb::kKvTabUnits / per_tok));
  const int grid = (n_tokens + tpc - 1) / tpc;
  rcb::kv_write_rope_tab_kernel<<<grid, rcb::kKvTabThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(q), q_stride, static_cast<const __nv_bfloat16*>(k),
      static_cast<const __nv_bfloat16*>(v), kv_stride, static_cast<__nv_bfloat16*>(q_out),
      positions_dev, slots_dev, n_tokens, n_q_heads, static_cast<__nv_bfloat16*>(kv_pool),
      block_tokens, block_elems, n_kv_heads, head_dim, layer,
      static_cast<const float4*>(rope_table_dev), tpc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rcb::set_cuda_error(e, "rcb_kv_write_rope_table");
  return RCB_OK;
}

extern "C" int rcb_kv_write_rope(const void* q, int64_t q_stride, const void* k, const void* v,
                                 int64_t kv_stride, void* q_out, const int32_t* positions_dev,
                                 const int32_t* slots_dev, int32_t n_tokens, int32_t n_q_heads,
                                 void* kv_pool, int32_t block_tokens, int32_t n_layers,
                                 int32_t n_kv_heads, int32_t head_dim, int32_t layer,
                                 float rope_theta, void* stream) {
  if (n_tokens == 0) return RCB_OK;
  if (head_dim % 16 != 0 || head_dim > 256 || layer < 0 || layer >= n_layers)
    return rcb::set_error(RCB_ERR_ARG, "head_dim must be a multiple of 16 (<= 256), layer in range");
  if (q_stride % 8 != 0 || kv_stride % 8 != 0)
    return rcb::set_error(RCB_ERR_ARG, "q/kv row strides must be multiples of 8 elements");
  const int64_t block_elems = int64_t(n_layers) * 2 * n_kv_heads * block_tokens * head_dim;
  rcb::kv_write_rope_kernel<<<n_tokens, rcb::kRopeThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(q), q_stride, static_cast<const __nv_bfloat16*>(k),
      static_cast<const __nv_bfloat16*>(v), kv_stride, static_cast<__nv_bfloat16*>(q_out),
      positions_dev, slots_dev, n_q_heads, static_cast<__nv_bfloat16*>(kv_pool), block_tokens,
      block_elems, n_kv_heads, head_dim, layer, log2f(rope_theta));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rcb::set_cuda_error(e, "rcb_kv_write_rope");
  return RCB_OK;
}
