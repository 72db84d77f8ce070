// tma_bench.cu -- diagnostics: TMA load throughput for halo-shaped boxes of
// an NHWC fp32 tensor (BASELINE C2 input, 16 x 64 x 64 x 64), 148 CTAs, each
// streaming its share of pixels through a 4-stage SMEM ring.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench scripts/tma_bench.cu -lcuda
// Variants (bytes per pixel row segment = one TMA request run):
//   0: box {8 fp32, R rows, 1}  x 8 chunks  (32-B segments, the old halo layout)
//   1: box {32 fp32, R rows}    x 2 halves  (128-B segments)
//   2: box {64 fp32, R rows}    x 1         (256-B segments)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(32) tma_stream(const __grid_constant__ CUtensorMap map, int variant,
                                                 int rows, long long pixels, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const long long per = (pixels + gridDim.x - 1) / gridDim.x;
  const long long p0 = per * blockIdx.x, p1 = min(pixels, p0 + per);
  const uint32_t stage_bytes = (uint32_t)rows * 256;
  unsigned long long t0 = clock64();
  int it = 0;
  for (int rep = 0; rep < 20; ++rep)
  for (long long p = p0; p < p1; p += rows, ++it) {
    const int s = it & 3;
    if (it >= 4) {  // wait for the load issued 4 iterations ago
      const uint32_t ph = ((it >> 2) - 1) & 1;
      asm volatile(
          "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(
              smem_u32(&bar[s])),
          "r"(ph));
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                 "r"(stage_bytes));
    const uint32_t dst = smem_u32(smem) + (uint32_t)s * stage_bytes;
    if (variant == 0) {
      for (int j = 0; j < 8; ++j)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                dst + (uint32_t)j * rows * 32),
            "l"(&map), "r"(smem_u32(&bar[s])), "r"(0), "r"((int)p), "r"(j));
    } else if (variant == 1) {
      for (int h = 0; h < 2; ++h)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                dst + (uint32_t)h * rows * 128),
            "l"(&map), "r"(smem_u32(&bar[s])), "r"(h * 32), "r"((int)p));
    } else {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              dst),
          "l"(&map), "r"(smem_u32(&bar[s])), "r"(0), "r"((int)p));
    }
  }
  for (int k = (it > 4 ? it - 4 : 0); k < it; ++k) {
    const int s = k & 3;
    const uint32_t ph = (k >> 2) & 1;
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(
            smem_u32(&bar[s])),
        "r"(ph));
  }
  cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

int main() {
  const long long pixels = 16LL * 64 * 64;
  const int cin = 64;
  float* x;
  cudaMalloc(&x, pixels * cin * 4);
  cudaMemset(x, 0, pixels * cin * 4);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  EncFn enc = (EncFn)f;
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const cuuint32_t es[3] = {1, 1, 1};
  for (int rows : {64, 128, 200}) {
    for (int v = 0; v < 3; ++v) {
      CUtensorMap m;
      CUresult rc;
      if (v == 0) {
        const cuuint64_t dims[3] = {8, (cuuint64_t)pixels, 8};
        const cuuint64_t str[2] = {(cuuint64_t)cin * 4, 32};
        const cuuint32_t box[3] = {8, (cuuint32_t)rows, 1};
        rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, str, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        const cuuint64_t dims[2] = {(cuuint64_t)cin, (cuuint64_t)pixels};
        const cuuint64_t str[1] = {(cuuint64_t)cin * 4};
        const cuuint32_t box[2] = {(cuuint32_t)(v == 1 ? 32 : 64), (cuuint32_t)rows};
        rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, str, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (rc != CUDA_SUCCESS) {
        printf("encode failed v=%d rows=%d rc=%d\n", v, rows, (int)rc);
        continue;
      }
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float best = 1e9f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        tma_stream<<<148, 32, 4 * rows * 256>>>(m, v, rows, pixels, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      cudaError_t e = cudaGetLastError();
      printf("rows=%3d variant %d (%3d-B segments): %.2f us, %.0f GB/s %s\n", rows, v,
             v == 0 ? 32 : v == 1 ? 128 : 256, best * 1e3, 20.0 * pixels * cin * 4 / (best * 1e-3) / 1e9,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
