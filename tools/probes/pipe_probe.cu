// Issue-rate probe for the softmax pipes on sm_100a: cycles per warp instruction for
// MUFU.EX2 (f32), ex2.approx.f16x2, FFMA2, FFMA, F2FP and mixes, with W warps per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cuda_fp16.h>

#define N_ITER 4096
#define CHAINS 8

template <int MODE>
__global__ void probe(float* out, long long* cyc) {
  float x[CHAINS];
  unsigned h[CHAINS];
  for (int i = 0; i < CHAINS; ++i) { x[i] = -0.001f * (threadIdx.x + i); h[i] = 0x3c003c00u + i; }
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      if (MODE == 0) {  // MUFU.EX2 f32
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      } else if (MODE == 1) {  // ex2.approx.f16x2
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      } else if (MODE == 2) {  // FFMA2
        unsigned long long v;
        asm volatile("mov.b64 %0, {%1, %1};" : "=l"(v) : "f"(x[i]));
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
        asm volatile("mov.b64 {%0, %0}, %1;" : "=f"(x[i]) : "l"(v));
      } else if (MODE == 3) {  // FFMA
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x[i]));
      } else if (MODE == 4) {  // 1 MUFU f32 + 3 FFMA
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
        float y = x[(i + 1) % CHAINS];
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(y));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(y));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(y));
        x[(i + 1) % CHAINS] = y;
      } else if (MODE == 5) {  // 1 f16x2 MUFU + 3 FFMA
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
        float y = x[i];
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(y));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(y));
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(y));
        x[i] = y;
      } else if (MODE == 6) {  // cvt f16x2 -> 2 f32
        float a, b;
        asm volatile("{.reg .b16 l, hh; mov.b32 {l, hh}, %2; cvt.f32.f16 %0, l; cvt.f32.f16 %1, hh;}" : "=f"(a), "=f"(b) : "r"(h[i]));
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(a), "f"(b));
      } else if (MODE == 7) {  // F2FP bf16 pack
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(x[i]), "f"(__uint_as_float(h[i])));
      } else if (MODE == 8) {  // ex2.approx.ftz.bf16x2
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < CHAINS; ++i) s += x[i] + __uint_as_float(h[i]);
  if (s == 12345.f) out[threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps_per_smsp, float* out, long long* cyc) {
  const int threads = 128 * warps_per_smsp;
  probe<MODE><<<148, threads>>>(out, cyc);
  probe<MODE><<<148, threads>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[64];
  cudaMemcpy(h, cyc, sizeof(long long) * (threads / 32), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int w = 0; w < threads / 32; ++w) mx = h[w] > mx ? h[w] : mx;
  const double per = mx / (double(N_ITER) * CHAINS);
  printf("%-28s warps/SMSP %d: %.2f cycles per (warp, loop body) -> %.2f per SMSP\n", name,
         warps_per_smsp, per, per / warps_per_smsp);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&cyc, 64 * 8);
  for (int w : {1, 2, 4}) {
    run<0>("MUFU.EX2 f32", w, out, cyc);
    run<1>("ex2.approx.f16x2", w, out, cyc);
    run<8>("ex2.approx.ftz.bf16x2", w, out, cyc);
    run<2>("FFMA2 (+movs)", w, out, cyc);
    run<3>("FFMA", w, out, cyc);
    run<4>("MUFU f32 + 3 FFMA", w, out, cyc);
    run<5>("MUFU f16x2 + 3 FFMA", w, out, cyc);
    run<6>("f16x2->2xf32->f16x2", w, out, cyc);
    run<7>("F2FP.BF16 pack", w, out, cyc);
  }
  return 0;
}
