// model_ops.cu — fused elementwise ops of the random-init decoder that prices
// ragsim's T(alpha, beta) and decode step on B200 (profile.py, timed.py).
//
// Not a ragsim stand-in by themselves: ragsim's interpolate (cost_model.py:106-117)
// and decode_ms_per_token (config.py:52) are priced by the WHOLE prefill of that
// model.  At a cached-prefix prefill (beta = 32) or a decode step (beta = 1) the
// per-layer fp32 residual / RMSNorm / SiLU chain ran as ~20 tiny torch kernels
// per layer, about as long as the weight-read-bound GEMMs; each chain is one
// kernel here.  Semantics match model.py's torch code: fp32 residual stream,
// h = bf16(x * rsqrt(mean(x^2) + eps) * w), a = bf16(silu(gate) * up).
#include <cuda_bf16.h>

#include "sm100.cuh"
#include "rcb_internal.h"

namespace rcb {
namespace {

constexpr int kNormThreads = 256;

__device__ __forceinline__ float bf(uint16_t v) { return __uint_as_float(uint32_t(v) << 16); }

// one CTA per row: x[row] (+= add[row]), h[row] = bf16(rmsnorm(x[row]) * w)
__global__ void __launch_bounds__(kNormThreads)
    rmsnorm_residual_kernel(float* __restrict__ x, const __nv_bfloat16* __restrict__ add,
                            const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ h,
                            int d, float eps) {
  const int64_t row = blockIdx.x;
  float4* xr = reinterpret_cast<float4*>(x + row * d);
  const uint2* ar = add != nullptr ? reinterpret_cast<const uint2*>(add + row * d) : nullptr;
  const int n4 = d / 4;
  float ss = 0.f;
  // pass 1: residual add (written back) and sum of squares; d <= 8192 -> <= 8 float4 per thread
  float4 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < n4) {
      float4 t = xr[i];
      if (ar != nullptr) {
        const uint2 a = ar[i];
        t.x += bf(a.x & 0xFFFF);
        t.y += bf(a.x >> 16);
        t.z += bf(a.y & 0xFFFF);
        t.w += bf(a.y >> 16);
        xr[i] = t;
      }
      v[k] = t;
      ss += t.x * t.x + t.y * t.y + t.z * t.z + t.w * t.w;
    }
  }
  __shared__ float red[kNormThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < kNormThreads / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / d + eps);
  const uint2* wr = reinterpret_cast<const uint2*>(w);
  uint2* hr = reinterpret_cast<uint2*>(h + row * d);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < n4) {
      const uint2 ww = __ldg(wr + i);
      const float4 t = v[k];
      uint2 o;
      o.x = pack_bf16(t.x * inv * bf(ww.x & 0xFFFF), t.y * inv * bf(ww.x >> 16));
      o.y = pack_bf16(t.z * inv * bf(ww.y & 0xFFFF), t.w * inv * bf(ww.y >> 16));
      hr[i] = o;
    }
  }
}

// a[t][j] = bf16(silu(gate) * up), gu = [T][2F] (gate = columns [0, F), up = [F, 2F))
__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ a,
                                int64_t n8, int f) {
  const int f8 = f / 8;
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < n8;
       u += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = u / f8;
    const int j = int(u - t * f8) * 8;
    const uint4 g = *reinterpret_cast<const uint4*>(gu + t * 2 * f + j);
    const uint4 p = *reinterpret_cast<const uint4*>(gu + t * 2 * f + f + j);
    const uint32_t gs[4] = {g.x, g.y, g.z, g.w}, ps[4] = {p.x, p.y, p.z, p.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float g0 = bf(gs[e] & 0xFFFF), g1 = bf(gs[e] >> 16);
      const float s0 = g0 / (1.f + __expf(-g0)), s1 = g1 / (1.f + __expf(-g1));
      o[e] = pack_bf16(s0 * bf(ps[e] & 0xFFFF), s1 * bf(ps[e] >> 16));
    }
    *reinterpret_cast<uint4*>(a + t * f + j) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace
}  // namespace rcb

extern "C" int rcb_rmsnorm_residual(float* x_dev, const void* add_dev, const void* weight_dev,
                                    void* h_out_dev, int32_t n_rows, int32_t d, float eps,
                                    void* stream) {
  if (n_rows < 0 || d <= 0 || d % 4 != 0 || d > 8 * 4 * rcb::kNormThreads)
    return rcb::set_error(RCB_ERR_ARG, "rmsnorm: d must be a positive multiple of 4, <= 8192");
  if (n_rows == 0) return RCB_OK;
  rcb::rmsnorm_residual_kernel<<<n_rows, rcb::kNormThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      x_dev, static_cast<const __nv_bfloat16*>(add_dev),
      static_cast<const __nv_bfloat16*>(weight_dev), static_cast<__nv_bfloat16*>(h_out_dev), d,
      eps);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rcb::set_cuda_error(e, "rcb_rmsnorm_residual");
  return RCB_OK;
}

extern "C" int rcb_silu_mul(const void* gate_up_dev, void* out_dev, int32_t n_rows, int32_t ffn,
                            void* stream) {
  if (n_rows < 0 || ffn <= 0 || ffn % 8 != 0)
    return rcb::set_error(RCB_ERR_ARG, "silu_mul: ffn must be a positive multiple of 8");
  if (n_rows == 0) return RCB_OK;
  const int64_t n8 = int64_t(n_rows) * (ffn / 8);
  const int64_t blocks = (n8 + 255) / 256;
  rcb::silu_mul_kernel<<<int(blocks < 4096 ? blocks : 4096), 256, 0,
                         static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(gate_up_dev), static_cast<__nv_bfloat16*>(out_dev), n8,
      ffn);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return rcb::set_cuda_error(e, "rcb_silu_mul");
  return RCB_OK;
}
