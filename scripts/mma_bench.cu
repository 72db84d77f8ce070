// mma_bench.cu -- diagnostics: tcgen05.mma (kind::f16, M=128, K=16) issue-to-
// completion throughput on one SM for different SMEM operand layouts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench scripts/mma_bench.cu
// Prints cycles per MMA for: no-swizzle K-major (aligned / 16-byte-offset
// start / power-of-two LBO) and 128B-swizzle K-major (aligned / row-offset
// start with base_offset), for N = 32, 64, 128, 256.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, int layout,
                                         int base_off) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) |
         ((uint64_t)(base_off & 7) << 49) | ((uint64_t)layout << 61);
}

__global__ void bench(int n, int variant, int iters, unsigned long long* out, int rot) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t a = smem_u32(smem), b = smem_u32(smem + 96 * 1024);
  uint64_t ad, bd;
  const int S = 200;
  switch (variant) {
    case 0: ad = desc(a, S * 16, 128, 0, 0); bd = desc(b, n * 16, 128, 0, 0); break;          // none, aligned
    case 1: ad = desc(a + 16, S * 16, 128, 0, 0); bd = desc(b, n * 16, 128, 0, 0); break;     // none, +16B
    case 2: ad = desc(a + 48, S * 16, 128, 0, 0); bd = desc(b, n * 16, 128, 0, 0); break;     // none, +48B
    case 3: ad = desc(a, 2048, 128, 0, 0); bd = desc(b, n * 16, 128, 0, 0); break;            // none, LBO 2048
    case 4: ad = desc(a, 16, 1024, 2, 0); bd = desc(b, 16, 1024, 2, 0); break;                // sw128 aligned
    case 5: ad = desc(a + 128, 16, 1024, 2, 1); bd = desc(b, 16, 1024, 2, 0); break;          // sw128 +1 row
    case 6: ad = desc(a + 640, 16, 1024, 2, 5); bd = desc(b, 16, 1024, 2, 0); break;          // sw128 +5 rows
    default: ad = desc(a, S * 16 + 16, 128, 0, 0); bd = desc(b, n * 16 + 16, 128, 0, 0); break; // none, odd LBO
  }
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  auto mma = [&](uint32_t d, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
  };
  unsigned long long t0 = 0;
  if (rot == 0) {  // thread 0 alone, one MMA per loop iteration
    if (threadIdx.x == 0) {
      t0 = clock64();
      for (int i = 0; i < iters; ++i) mma(tmem, i > 0);
    }
  } else if (rot == 1) {  // warp 0 uniform loop, elect.sync per MMA
    if (warp == 0) {
      t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        uint32_t pred;
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n" : "=r"(pred));
        if (pred) mma(tmem, i > 0);
        __syncwarp();
      }
    }
  } else {  // warp 0 elects once, the elected lane issues 8 MMAs per iteration (unrolled)
    if (warp == 0) {
      t0 = clock64();
      uint32_t pred;
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n" : "=r"(pred));
      if (pred) {
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
          for (int k = 0; k < 8; ++k) mma(tmem + (uint32_t)((k & 1) * n), (i + k) > 1);
        }
      }
      __syncwarp();
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
            smem_u32(&bar)));
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"none aligned", "none +16B", "none +48B", "none LBO2048",
                         "sw128 aligned", "sw128 +1row", "sw128 +5rows", "none odd-LBO"};
  const int iters = 4096;
  const char* modes[] = {"thread0", "warp+elect/mma", "elect-once unroll8"};
  for (int rot : {0, 1, 2}) {
    for (int n : {16, 32, 64, 128, 256}) {
      if (rot == 2 && n > 128) continue;
      for (int v : {0}) {
        bench<<<1, 128, 200 * 1024>>>(n, v, iters, d, rot);
        unsigned long long c = 0;
        cudaError_t e = cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        printf("%-20s N=%3d %-14s %7.1f cyc/mma  (floor %d)\n", modes[rot], n, names[v], (double)c / iters,
               128 * n / 256);
      }
    }
  }
  return 0;
}
