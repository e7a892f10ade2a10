// Verifies the tcgen05 16x256b load / 16x128b store register layouts used by the
// 4-threads-per-row softmax.  Writes TMEM with 32x32b (thread = lane, reg j = column j),
// reads back with 16x256b.x2 and reports (lane, column) of every register; then writes
// with 16x128b.x2 and reads back with 32x32b.
#include <cstdio>
#include <cstdint>

__global__ void k(int* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  if (warp == 0) {
    // value = lane * 1000 + column, columns 0..15
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = lane * 1000 + j;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(t), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                   "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    uint32_t r[8];
    // lanes 16..31 of the quadrant, columns 0..15 (x2 = two 8-column segments)
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(t + (16u << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) out[lane * 8 + j] = r[j];
    // store with 16x128b.x2 at lanes 0..15: value = 100000 + thread*100 + reg
    uint32_t w[4];
    for (int j = 0; j < 4; ++j) w[j] = 100000 + lane * 100 + j;
    asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1,%2,%3,%4};" ::"r"(t), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(t));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) out[256 + lane * 16 + j] = v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
}

int main() {
  int* d;
  cudaMalloc(&d, 4096 * 4);
  cudaMemset(d, 0xff, 4096 * 4);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  int h[4096];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("16x256b.x2 load at lane base 16: thread -> reg j = (lane, col)\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%2d:", t);
    for (int j = 0; j < 8; ++j) printf(" (%d,%d)", h[t * 8 + j] / 1000, h[t * 8 + j] % 1000);
    printf("\n");
  }
  printf("16x128b.x2 store at lane base 0: (lane, col) <- thread.reg\n");
  for (int l = 0; l < 16; ++l) {
    printf("lane %2d:", l);
    for (int c = 0; c < 8; ++c) {
      int v = h[256 + l * 16 + c];
      printf(" t%d.r%d", (v - 100000) / 100, (v - 100000) % 100);
    }
    printf("\n");
  }
  return 0;
}
