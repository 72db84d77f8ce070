// sw128_test.cu -- diagnostics: known-answer test of a row-shifted A operand
// in the 128-byte-swizzle K-major layout (bf16), the layout a TMA box
// {64 channels, rows} with CU_TENSOR_MAP_SWIZZLE_128B writes.  The halo-shift
// GEMM moves the A start by `shift` rows; this checks which descriptor
// base_offset makes that correct.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sw128_test scripts/sw128_test.cu
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, int layout,
                                         int base_off) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) |
         ((uint64_t)(base_off & 7) << 49) | ((uint64_t)layout << 61);
}

constexpr int ROWS = 160, K = 64, N = 64;

// A: ROWS x K bf16 (row-major host), B: N x K.  D = A[shift : shift+128] . B^T
__global__ void kat(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int shift, int bo_mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sa = smem;                 // SW128 K-major: row r at r*128, chunk c at (c ^ (r&7))*16
  uint8_t* sb = smem + ROWS * 128 + 1024 - (ROWS * 128) % 1024;  // no-swizzle [chunk][row][16B]
  for (int i = threadIdx.x; i < ROWS * K; i += blockDim.x) {
    const int r = i / K, k = i % K, c = k / 8;
    *reinterpret_cast<__nv_bfloat16*>(sa + r * 128 + ((c ^ (r & 7)) << 4) + (k % 8) * 2) = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + (k / 8) * N * 16 + n * 16 + (k % 8) * 2) = B[i];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint32_t a_addr = smem_u32(sa) + (uint32_t)shift * 128 + (uint32_t)ks * 32;
      const int bo = bo_mode == 0 ? 0 : (bo_mode == 1 ? (shift & 7) : ((a_addr >> 7) & 7));
      const uint64_t ad = desc(a_addr, 16, 1024, 2, bo);
      const uint64_t bd = desc(smem_u32(sb) + (uint32_t)ks * 2 * N * 16, N * 16, 128, 0, 0);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
              tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(ks ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int m = warp * 32 + lane;
  for (int c = 0; c < N; ++c) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                 : "=r"(r)
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    D[m * N + c] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  __nv_bfloat16 *hA = new __nv_bfloat16[ROWS * K], *hB = new __nv_bfloat16[N * K];
  srand(7);
  for (int i = 0; i < ROWS * K; ++i) hA[i] = __float2bfloat16((float)(rand() % 9 - 4));
  for (int i = 0; i < N * K; ++i) hB[i] = __float2bfloat16((float)(rand() % 9 - 4));
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, ROWS * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, hA, ROWS * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kat, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  float* hD = new float[128 * N];
  const char* modes[] = {"base_offset=0", "base_offset=shift&7", "base_offset=(addr>>7)&7"};
  int ok_any[3] = {1, 1, 1};
  for (int shift : {0, 1, 3, 7, 8, 17, 31}) {
    for (int bo = 0; bo < 3; ++bo) {
      cudaMemset(dD, 0, 128 * N * 4);
      kat<<<1, 128, 64 * 1024>>>(dA, dB, dD, shift, bo);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          float s = 0;
          for (int k = 0; k < K; ++k)
            s += __bfloat162float(hA[(m + shift) * K + k]) * __bfloat162float(hB[n * K + k]);
          bad += hD[m * N + n] != s;
        }
      if (bad || e != cudaSuccess) ok_any[bo] = 0;
      printf("shift %2d %-24s: %s mismatches %d\n", shift, modes[bo], cudaGetErrorString(e), bad);
    }
  }
  for (int bo = 0; bo < 3; ++bo) printf("MODE %s: %s\n", modes[bo], ok_any[bo] ? "ALL OK" : "FAILS");
  return 0;
}
