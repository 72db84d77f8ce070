// mma2_bench.cu -- diagnostics: tcgen05.mma.cta_group::2 (M = 256, K = 16,
// bf16, 128-byte swizzle K-major operands as the pair kernel uses them)
// throughput for N = 64 / 128 / 256, on one CTA pair, operands resident in
// shared memory (no loads).  Also times the same MMAs with a commit after
// every 4 (one pipeline stage) to see the commit cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma2 scripts/mma2_bench.cu && /tmp/mma2
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ bool elect() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "+r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(ph)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    bench(int n, int stages, int commit_every, unsigned long long* out, int spin) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2, done;
  __shared__ uint32_t tslot;
  const uint32_t rank = ctarank();
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done)) : "memory");  // phase 0 complete
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  // A: 4 stages x 16 KB (128 rows x 128 B), B: 4 stages x (n/2 rows x 128 B)
  const uint32_t a0 = smem_u32(smem), b0 = a0 + 64 * 1024;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (rank == 0 && warp == 0) {  // the whole warp runs the loop; one elected lane issues
    unsigned long long t0 = clock64();
    int c = 0;
    for (int s = 0; s < stages; ++s) {
      if (spin < 0) mbar_wait(&done, 0);  // a stage's barrier wait on a completed phase
      const uint64_t ad = sw128_desc(a0 + (uint32_t)(s & 3) * 16384);
      const uint64_t bd = sw128_desc(b0 + (uint32_t)(s & 3) * (n / 2) * 128);
      if (n > 0 && elect())
        for (int ks = 0; ks < 4; ++ks) mma2(tmem + (uint32_t)((s & 1) * n), ad + 2u * ks, bd + 2u * ks, idesc, ks ? 1u : 0u);
      if (spin > 0) {  // per-stage bookkeeping stand-in: does the MMA queue hide it?
        const unsigned long long ts = clock64();
        while (clock64() - ts < (unsigned long long)spin) {}
      }
      if (commit_every && ++c == commit_every) {
        c = 0;
        if (elect()) commit2(&bar2);
      }
      __syncwarp();
    }
    if (elect()) commit2(&bar);
    __syncwarp();
    if (threadIdx.x == 0) out[0] = t0;
  }
  if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);  // the final commit
    if (rank == 0) out[1] = clock64();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int n : {0, 128, 256})
    for (int spin : {0, -1})
      for (int ce : {0, 1}) {
        if (spin && !ce) continue;
        const int stages = 2000;
        bench<<<2, 128, 160 * 1024>>>(n, stages, ce, d, spin);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("N=%3d commit/stage=%d spin=%3d: %.1f cycles per stage of 4 MMAs (ideal %d) %s\n", n, ce, spin,
               (double)(h[1] - h[0]) / stages, 4 * 128 * n / 256, cudaGetErrorString(e));
      }
  return 0;
}
