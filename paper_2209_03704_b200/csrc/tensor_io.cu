#include <cmath>
// tensor_io.cu -- SGC1 tensor container (reference tensor_io.hpp:12-103), host
// side of the boundary: the format the reference's tools exchange tensors in
// (tools/segconv.cpp apply/verify read and write it).  Same header checks, error
// kinds and byte offsets as the reference; plus a batch loader that streams
// files into a pinned NHWC staging buffer and uploads each image as soon as it
// is read.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "kernels.h"
#include "segconv_b200.h"

namespace segconv_b200 {
segconv_status set_error(segconv_status st, const char* msg);  // capi.cu: segconv_last_error()

namespace {

thread_local size_t g_parse_offset = 0;

segconv_status parse_error(size_t offset, const std::string& msg) {
  g_parse_offset = offset;
  return set_error(SEGCONV_E_PARSE, (msg + " (byte offset " + std::to_string(offset) + ")").c_str());
}

uint32_t u32le(const unsigned char* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

void put_u32le(unsigned char* p, uint32_t v) {
  p[0] = (unsigned char)(v & 0xff);
  p[1] = (unsigned char)((v >> 8) & 0xff);
  p[2] = (unsigned char)((v >> 16) & 0xff);
  p[3] = (unsigned char)((v >> 24) & 0xff);
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

// reference tensor_io.hpp:53-74
segconv_status peek(const char* path, segconv_tensor_file_info* info) {
  if (!path || !info) return set_error(SEGCONV_E_CONTRACT, "null path or info pointer");
  File in;
  in.f = fopen(path, "rb");
  if (!in.f) return set_error(SEGCONV_E_IO, (std::string("cannot open ") + path).c_str());
  unsigned char hdr[20];
  const size_t got = fread(hdr, 1, sizeof hdr, in.f);
  if (got != sizeof hdr)
    return parse_error(got, std::string(path) + ": truncated header, expected 20 bytes, got " +
                                std::to_string(got));
  if (memcmp(hdr, "SGC1", 4) != 0) return parse_error(0, std::string(path) + ": bad magic");
  const uint32_t h = u32le(hdr + 4), w = u32le(hdr + 8), c = u32le(hdr + 12), prec = u32le(hdr + 16);
  if (prec > 1) return parse_error(16, std::string(path) + ": unknown precision tag " + std::to_string(prec));
  // the reference casts the u32 fields to int before the positivity check
  if ((int)h < 1 || (int)w < 1 || (int)c < 1)
    return parse_error(4, std::string(path) + ": non-positive dimension in header");
  info->height = (int)h;
  info->width = (int)w;
  info->channels = (int)c;
  info->precision = (int)prec;
  return SEGCONV_OK;
}

size_t elem_size(int dtype) { return dtype == SEGCONV_F64 ? 8 : 4; }

template <typename T>
bool all_finite(const T* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

// reference tensor_io.hpp:76-91; the payload is read straight into dst
segconv_status load(const char* path, segconv_dtype dtype, void* dst, size_t dst_bytes,
                    segconv_tensor_file_info* out_info) {
  segconv_tensor_file_info info;
  segconv_status st = peek(path, &info);
  if (st != SEGCONV_OK) return st;
  if (dtype != SEGCONV_F32 && dtype != SEGCONV_F64)
    return set_error(SEGCONV_E_CONTRACT, "SGC1 stores f32 or f64 tensors");
  if (info.precision != (dtype == SEGCONV_F64 ? 1 : 0))
    return set_error(SEGCONV_E_CONTRACT,
                     (std::string(path) + ": stored precision does not match requested element type").c_str());
  const size_t count = (size_t)info.height * info.width * info.channels;
  const size_t expect = 20 + count * elem_size(dtype);
  File in;
  in.f = fopen(path, "rb");
  if (!in.f) return set_error(SEGCONV_E_IO, (std::string("cannot open ") + path).c_str());
  if (fseek(in.f, 0, SEEK_END) != 0) return set_error(SEGCONV_E_IO, (std::string("read failure on ") + path).c_str());
  const long len = ftell(in.f);
  if (len < 0) return set_error(SEGCONV_E_IO, (std::string("read failure on ") + path).c_str());
  if ((size_t)len != expect)
    return parse_error((size_t)len < expect ? (size_t)len : expect,
                       std::string(path) + ": payload size mismatch, expected " + std::to_string(expect) +
                           " bytes total, got " + std::to_string(len));
  if (!dst || dst_bytes < count * elem_size(dtype))
    return set_error(SEGCONV_E_CONTRACT, "destination buffer is too small");
  if (fseek(in.f, 20, SEEK_SET) != 0 || fread(dst, 1, count * elem_size(dtype), in.f) != count * elem_size(dtype))
    return set_error(SEGCONV_E_IO, (std::string("read failure on ") + path).c_str());
  // the reference builds the result through Tensor::from_data, which rejects
  // non-finite payloads (tensor.hpp:87-88)
  const bool finite = dtype == SEGCONV_F64 ? all_finite((const double*)dst, count)
                                           : all_finite((const float*)dst, count);
  if (!finite) return set_error(SEGCONV_E_CONTRACT, "tensor data contains a non-finite element");
  if (out_info) *out_info = info;
  return SEGCONV_OK;
}

}  // namespace
}  // namespace segconv_b200

using namespace segconv_b200;

extern "C" {

size_t segconv_last_error_offset(void) { return g_parse_offset; }

segconv_status segconv_peek_tensor_file(const char* path, segconv_tensor_file_info* info) {
  return peek(path, info);
}

segconv_status segconv_load_tensor(const char* path, segconv_dtype dtype, void* host_dst, size_t dst_bytes) {
  return load(path, dtype, host_dst, dst_bytes, nullptr);
}

segconv_status segconv_save_tensor(const char* path, const void* host_src, int height, int width, int channels,
                                   segconv_dtype dtype) {
  if (!path) return set_error(SEGCONV_E_CONTRACT, "null path");
  if (dtype != SEGCONV_F32 && dtype != SEGCONV_F64)
    return set_error(SEGCONV_E_CONTRACT, "SGC1 stores f32 or f64 tensors");
  if (height < 0 || width < 0 || channels < 0) return set_error(SEGCONV_E_SHAPE, "negative tensor dimension");
  const size_t bytes = (size_t)height * width * channels * elem_size(dtype);
  if (bytes && !host_src) return set_error(SEGCONV_E_CONTRACT, "null source pointer");
  File out;
  out.f = fopen(path, "wb");
  if (!out.f) return set_error(SEGCONV_E_IO, (std::string("cannot open ") + path + " for writing").c_str());
  unsigned char hdr[20];
  memcpy(hdr, "SGC1", 4);
  put_u32le(hdr + 4, (uint32_t)height);
  put_u32le(hdr + 8, (uint32_t)width);
  put_u32le(hdr + 12, (uint32_t)channels);
  put_u32le(hdr + 16, dtype == SEGCONV_F64 ? 1u : 0u);
  if (fwrite(hdr, 1, 20, out.f) != 20 || (bytes && fwrite(host_src, 1, bytes, out.f) != bytes) ||
      fflush(out.f) != 0)
    return set_error(SEGCONV_E_IO, (std::string("write failure on ") + path).c_str());
  return SEGCONV_OK;
}

segconv_status segconv_load_tensor_batch(const char* const* paths, int count, segconv_dtype dtype,
                                         void* host_staging, void* d_dst, void* stream) {
  if (count < 0 || (count > 0 && (!paths || !host_staging)))
    return set_error(SEGCONV_E_CONTRACT, "bad batch arguments");
  if (count == 0) return SEGCONV_OK;
  segconv_tensor_file_info first;
  segconv_status st = peek(paths[0], &first);
  if (st != SEGCONV_OK) return st;
  const size_t img = (size_t)first.height * first.width * first.channels * elem_size(dtype);
  cudaStream_t s = (cudaStream_t)stream;
  for (int i = 0; i < count; ++i) {
    segconv_tensor_file_info info;
    char* slot = (char*)host_staging + (size_t)i * img;
    st = load(paths[i], dtype, slot, img, &info);
    if (st != SEGCONV_OK) return st;
    if (info.height != first.height || info.width != first.width || info.channels != first.channels)
      return set_error(SEGCONV_E_CONTRACT,
                       (std::string(paths[i]) + ": shape differs from the first file of the batch").c_str());
    if (d_dst) {
      const cudaError_t e = cudaMemcpyAsync((char*)d_dst + (size_t)i * img, slot, img, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return set_error(SEGCONV_E_CUDA, cudaGetErrorString(e));
    }
  }
  return SEGCONV_OK;
}

}  // extern "C"
