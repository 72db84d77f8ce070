// launch_overhead.cu -- diagnostics: device time of near-empty kernels shaped
// like the tile / pair kernels (296 x 320 threads), with and without large
// dynamic shared memory and a TMEM alloc / dealloc, to find where a kernel's
// duration outside every CTA's lifetime goes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lo scripts/launch_overhead.cu && /tmp/lo
//   (and under ncu --metrics gpu__time_duration.sum,sm__cycles_active.max)
#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(320, 2) k_empty(int* out) {
  extern __shared__ uint8_t smem[];
  if (threadIdx.x == 0 && out) out[blockIdx.x] = 1;
}

__global__ void __launch_bounds__(320, 2) k_tmem(int* out, long long* clk) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  long long t0 = clock64(), t1 = 0, t2 = 0, t3 = 0;
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    t1 = clock64();
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    t2 = clock64();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0 && out) out[blockIdx.x] = slot;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 8) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const long long t4 = clock64();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(slot));
    t3 = clock64();
    if ((threadIdx.x & 31) == 0 && clk) {
      clk[blockIdx.x * 4 + 0] = t1 - t0;
      clk[blockIdx.x * 4 + 1] = t2 - t1;
      clk[blockIdx.x * 4 + 2] = t4 - t2;
      clk[blockIdx.x * 4 + 3] = t3 - t4;
    }
  }
}

int main() {
  int* d;
  cudaMalloc(&d, 4096 * 4);
  long long* clk;
  cudaMalloc(&clk, 296 * 4 * 8);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
  cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 113 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int var = 0; var < 4; ++var) {
    const size_t smem = (var & 1) ? 103 * 1024 : 0;
    float best = 1e9f;
    for (int it = 0; it < 20; ++it) {
      cudaEventRecord(a);
      if (var < 2)
        k_empty<<<296, 320, smem>>>(d);
      else
        k_tmem<<<296, 320, smem>>>(d, clk);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 2 && ms < best) best = ms;
    }
    printf("%s smem %6zu: best %.2f us (events around one launch)\n", var < 2 ? "empty" : "tmem ", smem,
           best * 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  long long h[296 * 4];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  for (int c : {0, 1, 100, 147, 148, 200, 295})
    printf("CTA %3d: alloc %lld relinquish %lld body %lld dealloc %lld cycles\n", c, h[c * 4], h[c * 4 + 1],
           h[c * 4 + 2], h[c * 4 + 3]);
  return 0;
}
