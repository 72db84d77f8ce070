// tmem_a_test.cu -- diagnostics: tcgen05.mma kind::f16 with the A operand in
// TMEM (the "ts" form), cta_group::1, M=128, K=16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_a_test scripts/tmem_a_test.cu
// 1. Known-answer test of the TMEM A layout assumed by tc_fold.cu's TMEM-A
//    variant: lane m = row m, column c holds the fp16 pair (A[m][2c], A[m][2c+1]),
//    so one K=16 step occupies 8 consecutive columns.
// 2. Issue-to-completion cycles per MMA for N = 64, 128, 256 (A in TMEM, B in
//    SMEM no-swizzle K-major) against the SS form.
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);  // fp16 A/B
}

// A: 128 x KS*16 halves row-major; B: N x KS*16 halves row-major; D out: 128 x N floats.
__global__ void kat(const __half* A, const __half* B, float* D, int N, int KS, int ts) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = KS * 16;
  uint8_t* sa = smem;              // A in SMEM (SS form): [chunk][row 128][16 B]
  uint8_t* sb = smem + 128 * K * 2;  // B: [chunk][row N][16 B]
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    *reinterpret_cast<__half*>(sa + (k / 8) * 128 * 16 + m * 16 + (k % 8) * 2) = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__half*>(sb + (k / 8) * N * 16 + n * 16 + (k % 8) * 2) = B[i];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t a_col = 256;  // A lives in columns [256, 256 + KS*8)
  // A -> TMEM: warp w writes lanes 32w..32w+31, 8 columns per K=16 step
  {
    const int m = warp * 32 + lane;
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t r[8];
      for (int c = 0; c < 8; ++c) {
        const __half lo = A[m * K + ks * 16 + 2 * c], hi = A[m * K + ks * 16 + 2 * c + 1];
        r[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + a_col + ks * 8;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    for (int ks = 0; ks < KS; ++ks) {
      const uint64_t bd = desc(smem_u32(sb) + ks * 2 * N * 16, N * 16, 128);
      const uint32_t acc = ks ? 1u : 0u;
      if (ts) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
            "r"(tmem + a_col + ks * 8), "l"(bd), "r"(idesc(N)), "r"(acc));
      } else {
        const uint64_t ad = desc(smem_u32(sa) + ks * 2 * 128 * 16, 128 * 16, 128);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc(N)), "r"(acc));
      }
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Throughput: iters MMAs back to back (A TMEM or SMEM), cycling over nd
// independent accumulators (nd = 1: every MMA depends on the previous one).
__global__ void thr(int N, int iters, int ts, int nd, int fmt, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint64_t bd = desc(smem_u32(smem + 16384), N * 16, 128);
    const uint64_t ad = desc(smem_u32(smem), 128 * 16, 128);
    const uint32_t a_tm = tmem + 448;  // A columns [448, 512)
    const uint32_t dstride = nd == 1 ? 0u : (uint32_t)(448 / nd) & ~7u;
    const uint32_t id = idesc(N) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t d = tmem + (uint32_t)(k % nd) * dstride;
        if (ts)
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n" ::"r"(d),
                       "r"(a_tm + (uint32_t)(k & 7) * 8), "l"(bd), "r"(id));
        else
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(d),
                       "l"(ad), "l"(bd), "r"(id));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
            smem_u32(&bar)));
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// The C2 fold kernel's MMA stream: per unit 2 stages x 4 shifts x 2 k-steps x
// 3 split MMAs (N=128, A in TMEM), B = halo columns (COL = S_pad*16 bytes,
// LBO = 2*COL), B start moved by shift*16 bytes.  variant bit0: zero the
// shift offsets; bit1: LBO = 2048 (compact B); bit2: SS form (A in SMEM).
__global__ void fold_stream(int units, int variant, unsigned long long* out) {
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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if ((variant & 8) ? warp == 0 : threadIdx.x == 0) {
    const uint32_t COL = (variant & 2) ? 2048 / 2 : 200 * 16;
    const uint32_t LBO = 2 * COL;
    const int shift_off[4] = {0, 1, 64, 65};
    const uint32_t x0 = smem_u32(smem);
    const uint32_t id = idesc(128);
    unsigned long long t0 = clock64();
    for (int u = 0; u < units; ++u) {
      const uint32_t d = tmem + (uint32_t)(u & 1) * 128;
      for (int kb = 0; kb < 2; ++kb) {
        const uint32_t xa = x0 + (uint32_t)kb * 4 * LBO;
        for (int s = 0; s < 4; ++s) {
          const uint32_t xs = xa + ((variant & 1) ? 0u : (uint32_t)shift_off[s] * 16);
          for (int ks = 0; ks < 2; ++ks) {
            const uint32_t acc = (kb == 0 && s == 0 && ks == 0) ? 0u : 1u;
            const uint32_t xk = xs + (uint32_t)ks * 2 * LBO;
            const uint64_t xh = desc(xk, LBO, 128), xl = desc(xk + COL, LBO, 128);
            const uint32_t wh = tmem + 256 + (uint32_t)((s * 2 * 4 + kb * 2 + ks) * 8);
            const uint32_t wl = wh + 32;
            if (variant & 8) {
#define MMA_E(A_, B_, ACC_) asm volatile("{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(A_), "l"(B_), "r"(id), "r"(ACC_))
              MMA_E(wh, xh, acc);
              MMA_E(wl, xh, 1u);
              MMA_E(wh, xl, 1u);
            } else if (variant & 4) {
              const uint64_t ah = desc(x0 + 100 * 1024 + (uint32_t)(s * 2 + ks) * 4096, 2048, 128);
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(ah), "l"(xh), "r"(id), "r"(acc));
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(ah + 64), "l"(xh), "r"(id), "r"(1u));
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(ah), "l"(xl), "r"(id), "r"(1u));
            } else {
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(wh), "l"(xh), "r"(id), "r"(acc));
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(wl), "l"(xh), "r"(id), "r"(1u));
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(wh), "l"(xl), "r"(id), "r"(1u));
            }
          }
        }
      }
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
        smem_u32(&bar)));
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
            smem_u32(&bar)));
    if (threadIdx.x == 0) out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  int fails = 0;
  for (int N : {64, 128, 256}) {
    const int KS = 4, K = KS * 16;
    __half *hA = new __half[128 * K], *hB = new __half[N * K];
    float* ref = new float[128 * N];
    srand(N);
    for (int i = 0; i < 128 * K; ++i) hA[i] = __float2half((float)(rand() % 9 - 4));
    for (int i = 0; i < N * K; ++i) hB[i] = __float2half((float)(rand() % 9 - 4));
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        float s = 0;
        for (int k = 0; k < K; ++k) s += __half2float(hA[m * K + k]) * __half2float(hB[n * K + k]);
        ref[m * N + n] = s;
      }
    __half *dA, *dB;
    float* dD;
    cudaMalloc(&dA, 128 * K * 2);
    cudaMalloc(&dB, N * K * 2);
    cudaMalloc(&dD, 128 * N * 4);
    cudaMemcpy(dA, hA, 128 * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(kat, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int ts = 0; ts < 2; ++ts) {
      cudaMemset(dD, 0, 128 * N * 4);
      kat<<<1, 128, 100 * 1024>>>(dA, dB, dD, N, KS, ts);
      cudaError_t e = cudaDeviceSynchronize();
      float* hD = new float[128 * N];
      cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < 128 * N; ++i) bad += hD[i] != ref[i];
      printf("KAT N=%d %s: %s, mismatches %d / %d (D[0]=%g ref %g, D[5*N+3]=%g ref %g)\n", N,
             ts ? "A-in-TMEM" : "SS", cudaGetErrorString(e), bad, 128 * N, hD[0], ref[0],
             hD[5 * N + 3], ref[5 * N + 3]);
      fails += bad != 0 || e != cudaSuccess;
      delete[] hD;
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  unsigned long long* dout;
  cudaMalloc(&dout, 8);
  cudaFuncSetAttribute(thr, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int fmt = 0; fmt < 2; ++fmt)
    for (int N : {64, 128, 256})
      for (int ts = 0; ts < 2; ++ts)
        for (int nd : {1, 2}) {
          if (N * nd > 448) continue;
          const int iters = 4096;
          thr<<<1, 128, 64 * 1024>>>(N, iters, ts, nd, fmt, dout);
          thr<<<1, 128, 64 * 1024>>>(N, iters, ts, nd, fmt, dout);
          unsigned long long c = 0;
          cudaMemcpy(&c, dout, 8, cudaMemcpyDeviceToHost);
          printf("THR %s N=%3d %s accumulators=%d: %.1f cycles/MMA (ideal N/2 = %d)\n",
                 fmt ? "bf16" : "fp16", N, ts ? "TS" : "SS", nd, (double)c / iters, N / 2);
        }
  cudaFuncSetAttribute(fold_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int v : {0, 4, 8, 9}) {
    const int units = 64;
    fold_stream<<<1, 128, 200 * 1024>>>(units, v, dout);
    fold_stream<<<1, 128, 200 * 1024>>>(units, v, dout);
    unsigned long long c = 0;
    cudaMemcpy(&c, dout, 8, cudaMemcpyDeviceToHost);
    printf("FOLD variant %d (%s%s%s): %.1f cycles/MMA, %.0f cycles/unit (ideal 64/MMA)\n", v,
           (v & 8) ? "TS warp-uniform" : (v & 4) ? "SS" : "TS", (v & 1) ? " no-shift" : " shifted", (v & 2) ? " LBO2048" : " LBO6400",
           (double)c / (units * 48), (double)c / units);
  }
  printf(fails ? "KAT FAILED\n" : "KAT OK\n");
  return fails ? 1 : 0;
}
