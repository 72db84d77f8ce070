// common.cuh -- shared device helpers for the segconv B200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "segconv_b200.h"

namespace segconv_b200 {

// ------------------------------------------------------- per-device state
// Function attributes (dynamic shared memory size, cluster flags) and SM
// counts are properties of a device, and one process may drive several GPUs
// (the multi-GPU stack driver does, from one thread per device).  Each launch
// site keeps one PerDeviceOnce per kernel instantiation: the setup runs once
// per device id, lock-free; a concurrent duplicate run is harmless (the
// attributes are idempotent).
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  template <class F>
  cudaError_t run(F&& f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = f();
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
  }
};

// SM count of the current device (cached per device id; 148 on B200).
inline int device_sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  int v = cache[dev & 63].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  cache[dev & 63].store(v, std::memory_order_relaxed);
  return v;
}

// Sets the kernel's dynamic shared memory limit once per device.
template <typename K>
inline cudaError_t smem_attr_once(PerDeviceOnce& once, K kern, int bytes) {
  return once.run([&] {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  });
}

// ----------------------------------------------------------------- dtypes
template <typename T>
struct DT;
template <>
struct DT<float> {
  static constexpr int id = SEGCONV_F32;
};
template <>
struct DT<double> {
  static constexpr int id = SEGCONV_F64;
};
template <>
struct DT<__nv_bfloat16> {
  static constexpr int id = SEGCONV_BF16;
};

__device__ __forceinline__ float to_acc(float v) { return v; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ double to_acc(double v) { return v; }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ double from_f<double>(float v) { return (double)v; }

template <typename T>
__device__ __forceinline__ T from_d(double v);
template <>
__device__ __forceinline__ double from_d<double>(double v) { return v; }
template <>
__device__ __forceinline__ float from_d<float>(double v) { return (float)v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_d<__nv_bfloat16>(double v) {
  return __float2bfloat16_rn((float)v);
}

// 32-byte global accesses (sm_100 STG.E.256 / LDG.E.256); the address must be
// 32-byte aligned.  Epilogues writing one anchor's features per thread are
// bound by the number of scattered store instructions, so wider is faster.
__device__ __forceinline__ void st_global_v8(void* ptr, const uint32_t* w) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ptr), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
__device__ __forceinline__ void st_global_v8f(float* ptr, const float* v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(ptr), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void ld_global_v8f(const float* ptr, float* v) {
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(ptr)
               : "memory");
}
__device__ __forceinline__ bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }

// --------------------------------------------------------------- epilogue
// Order: + bias[f], then ReLU or tanh (SEGCONV_EPI_* flags).
__device__ __forceinline__ float epilogue_apply(float v, unsigned epi, const float* bias, int f) {
  if (epi & SEGCONV_EPI_BIAS) v += __ldg(bias + f);
  if (epi & SEGCONV_EPI_RELU) v = fmaxf(v, 0.0f);
  if (epi & SEGCONV_EPI_TANH) v = tanhf(v);
  return v;
}
__device__ __forceinline__ double epilogue_apply(double v, unsigned epi, const float* bias, int f) {
  if (epi & SEGCONV_EPI_BIAS) v += (double)__ldg(bias + f);
  if (epi & SEGCONV_EPI_RELU) v = v > 0.0 ? v : 0.0;
  if (epi & SEGCONV_EPI_TANH) v = tanh(v);
  return v;
}

// Store with the runtime output dtype (warp-uniform branch).
__device__ __forceinline__ void store_out(void* y, long long idx, float v, int y_dtype) {
  if (y_dtype == SEGCONV_BF16)
    reinterpret_cast<__nv_bfloat16*>(y)[idx] = __float2bfloat16_rn(v);
  else if (y_dtype == SEGCONV_F64)
    reinterpret_cast<double*>(y)[idx] = (double)v;
  else
    reinterpret_cast<float*>(y)[idx] = v;
}
__device__ __forceinline__ void store_out(void* y, long long idx, double v, int y_dtype) {
  if (y_dtype == SEGCONV_BF16)
    reinterpret_cast<__nv_bfloat16*>(y)[idx] = __float2bfloat16_rn((float)v);
  else if (y_dtype == SEGCONV_F64)
    reinterpret_cast<double*>(y)[idx] = v;
  else
    reinterpret_cast<float*>(y)[idx] = (float)v;
}

}  // namespace segconv_b200
