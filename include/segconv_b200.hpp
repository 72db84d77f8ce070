// segconv_b200.hpp -- drop-in C++ host API with the reference's operator names.
//
// Replace `#include "segconv.hpp"` (reference proj/include/segconv.hpp:8-22)
// with `#include "segconv_b200.hpp"` and link libsegconv_b200.so + cudart.
// The names, argument meaning, layouts (HWC tensors, (kh,kw,cin,cout)
// kernels) and exceptions (ShapeError / ContractError) are the reference's;
// the arithmetic runs in the sm_100a kernels behind include/segconv_b200.h.
// Calls take host tensors (value semantics, like the reference): each op
// copies its inputs to the device, launches, and copies the result back.
// Batched / device-resident work should call the C ABI directly.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "segconv_b200.h"

namespace segconv {

// ------------------------------------------------------------- errors
// reference errors.hpp:10-41
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
  using Error::Error;
};
struct ContractError : Error {
  using Error::Error;
};
struct CudaError : Error {
  using Error::Error;
};
struct ParseError : Error {
  ParseError(const std::string& msg, std::size_t offset) : Error(msg), byte_offset(offset) {}
  std::size_t byte_offset;
};
struct IoError : Error {
  using Error::Error;
};
struct StateError : Error {
  using Error::Error;
};

inline void throw_on(segconv_status st) {
  if (st == SEGCONV_OK) return;
  const std::string msg = segconv_last_error();
  if (st == SEGCONV_E_SHAPE) throw ShapeError(msg);
  if (st == SEGCONV_E_CONTRACT) throw ContractError(msg);
  if (st == SEGCONV_E_PARSE) throw ParseError(msg, segconv_last_error_offset());
  if (st == SEGCONV_E_IO) throw IoError(msg);
  throw CudaError(msg);
}

template <typename T>
struct dtype_of;
template <>
struct dtype_of<float> {
  static constexpr segconv_dtype value = SEGCONV_F32;
};
template <>
struct dtype_of<double> {
  static constexpr segconv_dtype value = SEGCONV_F64;
};

// ------------------------------------------------------------- tensors
// HWC, channel innermost (reference tensor.hpp:57-145)
template <typename T>
class Tensor {
  static_assert(std::is_floating_point_v<T>, "Tensor requires float or double");

 public:
  Tensor() = default;
  Tensor(int h, int w, int c) : h_(h), w_(w), c_(c) {
    if (h < 1 || w < 1 || c < 1)
      throw ShapeError("tensor dims must be positive, got " + std::to_string(h) + "x" +
                       std::to_string(w) + "x" + std::to_string(c));
    data_.assign(size(), T(0));
  }
  static Tensor from_data(int h, int w, int c, std::vector<T> values) {
    Tensor t(h, w, c);
    if (values.size() != t.size()) throw ContractError("tensor data length does not match dims");
    for (const T v : values)
      if (!std::isfinite(v)) throw ContractError("tensor data contains a non-finite element");
    t.data_ = std::move(values);
    return t;
  }
  int height() const { return h_; }
  int width() const { return w_; }
  int channels() const { return c_; }
  size_t size() const { return (size_t)h_ * w_ * c_; }
  T operator()(int i, int j, int ch) const { return data_[((size_t)i * w_ + j) * c_ + ch]; }
  T& operator()(int i, int j, int ch) { return data_[((size_t)i * w_ + j) * c_ + ch]; }
  const T* data() const { return data_.data(); }
  T* data() { return data_.data(); }
  bool same_shape(const Tensor& o) const { return h_ == o.h_ && w_ == o.w_ && c_ == o.c_; }

 private:
  int h_ = 0, w_ = 0, c_ = 0;
  std::vector<T> data_;
};

// (kh, kw, cin, cout), cout innermost (reference tensor.hpp:152-217)
template <typename T>
class Kernel {
 public:
  Kernel() = default;
  Kernel(int kh, int kw, int cin, int cout) : kh_(kh), kw_(kw), cin_(cin), cout_(cout) {
    if (kh < 0 || kw < 0 || cin < 1 || cout < 1) throw ShapeError("bad kernel dims");
    data_.assign(size(), T(0));
  }
  static Kernel from_data(int kh, int kw, int cin, int cout, std::vector<T> values) {
    if (kh < 1 || kw < 1 || cin < 1 || cout < 1) throw ShapeError("bad kernel dims");
    Kernel k(kh, kw, cin, cout);
    if (values.size() != k.size()) throw ContractError("kernel data length does not match dims");
    for (const T v : values)
      if (!std::isfinite(v)) throw ContractError("kernel data contains a non-finite element");
    k.data_ = std::move(values);
    return k;
  }
  int kh() const { return kh_; }
  int kw() const { return kw_; }
  int cin() const { return cin_; }
  int cout() const { return cout_; }
  size_t size() const { return (size_t)kh_ * kw_ * cin_ * cout_; }
  bool spatially_empty() const { return kh_ == 0 || kw_ == 0; }
  T operator()(int u, int v, int ch, int f) const {
    return data_[(((size_t)u * kw_ + v) * cin_ + ch) * cout_ + f];
  }
  T& operator()(int u, int v, int ch, int f) {
    return data_[(((size_t)u * kw_ + v) * cin_ + ch) * cout_ + f];
  }
  const T* data() const { return data_.data(); }
  T* data() { return data_.data(); }

 private:
  int kh_ = 0, kw_ = 0, cin_ = 0, cout_ = 0;
  std::vector<T> data_;
};

// ------------------------------------------------------------- device memory
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes) : n_(bytes) {
    if (bytes && cudaMalloc(&p_, bytes) != cudaSuccess) throw CudaError("cudaMalloc failed");
  }
  DeviceBuffer(const void* host, size_t bytes) : DeviceBuffer(bytes) {
    if (bytes && cudaMemcpy(p_, host, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
      throw CudaError("cudaMemcpy H2D failed");
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  void* get() const { return p_; }
  void to_host(void* dst, size_t bytes) const {
    if (cudaMemcpy(dst, p_, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      throw CudaError("cudaMemcpy D2H failed");
  }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

namespace detail {
// Value-semantics calls stage their host tensors through thread-local,
// grow-only device buffers (one per role), so a loop of per-image calls does
// not pay a cudaMalloc / cudaFree per tensor.
class Staged {
 public:
  Staged(int slot, size_t bytes) : p_(buffer(slot, bytes)) {}
  Staged(int slot, const void* host, size_t bytes) : Staged(slot, bytes) {
    if (bytes && cudaMemcpy(p_, host, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
      throw CudaError("cudaMemcpy H2D failed");
  }
  void* get() const { return p_; }
  void to_host(void* dst, size_t bytes) const {
    if (bytes && cudaMemcpy(dst, p_, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      throw CudaError("cudaMemcpy D2H failed");
  }

 private:
  static void* buffer(int slot, size_t bytes) {
    struct Slot {
      DeviceBuffer buf;
      size_t cap = 0;
    };
    thread_local Slot slots[8];
    Slot& s = slots[slot];
    if (s.cap < bytes) {
      s.buf = DeviceBuffer(bytes);
      s.cap = bytes;
    }
    return s.buf.get();
  }
  void* p_;
};
}  // namespace detail

// ------------------------------------------------------------- geometry
// reference geometry.hpp:18-53
struct TConvGeometry {
  int n_in = 0, kh = 0, kw = 0, p_orig = 0, p_fused = 0, up_h = 0, up_w = 0, out_h = 0, out_w = 0;
  bool trim_extra_row = false, trim_extra_col = false;
  segconv_geometry c() const {
    return {n_in, kh, kw, p_orig, p_fused, up_h, up_w, out_h, out_w, trim_extra_row, trim_extra_col};
  }
};

inline TConvGeometry tconv_geometry(int n_in, int kh, int kw, int p_orig) {
  segconv_geometry g;
  throw_on(segconv_tconv_geometry(n_in, kh, kw, p_orig, &g));
  return {g.n_in, g.kh, g.kw, g.p_orig, g.p_fused, g.up_h, g.up_w, g.out_h, g.out_w,
          g.trim_extra_row != 0, g.trim_extra_col != 0};
}
// reference segregation.hpp:23-36
inline int first_active_tap(int p, int r) { return segconv_first_active_tap(p, r); }
inline int active_tap_count(int n, int p, int r) { return segconv_active_tap_count(n, p, r); }
inline int class_input_offset(int p, int r) { return segconv_class_input_offset(p, r); }

// ------------------------------------------------------------- segregation
// Device counterpart of SubKernelSet<T> (reference segregation.hpp:43-55).
template <typename T>
struct SubKernelSet {
  segconv_subkernels desc{};
  std::shared_ptr<DeviceBuffer> panels;
  int source_kh = 0, source_kw = 0, p_orig_parity = 0;
  int cin() const { return desc.cin; }
  int cout() const { return desc.cout; }
  std::pair<int, int> offset(int r, int c) const {
    return {desc.off_r[r * 2 + c], desc.off_c[r * 2 + c]};
  }
};

// reference segregation.hpp:61-89.  `math` picks the consumer kernel
// (SEGCONV_MATH_AUTO: tensor cores where the layer suits them).
template <typename T>
SubKernelSet<T> segregate(const Kernel<T>& k, int p_orig, segconv_math math = SEGCONV_MATH_AUTO) {
  if (k.spatially_empty()) throw ContractError("cannot segregate a spatially empty kernel");
  if (p_orig < 0) throw ContractError("padding must be non-negative");
  SubKernelSet<T> s;
  throw_on(segconv_subkernels_for_math(k.kh(), k.kw(), k.cin(), k.cout(), p_orig,
                                       dtype_of<T>::value, math, &s.desc));
  const size_t esz = s.desc.dtype == SEGCONV_F64 ? 8 : s.desc.dtype == SEGCONV_F32 ? 4 : 2;
  s.panels = std::make_shared<DeviceBuffer>(std::max<size_t>(1, s.desc.total_elems * esz));
  detail::Staged dk(0, k.data(), k.size() * sizeof(T));
  throw_on(segconv_segregate(dk.get(), dtype_of<T>::value, &s.desc, s.panels->get(), nullptr));
  if (cudaDeviceSynchronize() != cudaSuccess) throw CudaError("segregate failed");
  s.source_kh = k.kh();
  s.source_kw = k.kw();
  s.p_orig_parity = p_orig & 1;
  return s;
}

// ------------------------------------------------------------- operators
// reference fused_tconv.hpp:69-82
template <typename T>
Tensor<T> transpose_conv_fused(const Tensor<T>& input, const SubKernelSet<T>& sks,
                               const TConvGeometry& geom) {
  if (input.height() != geom.n_in || input.width() != geom.n_in)
    throw ContractError("input size does not match the geometry");
  Tensor<T> out(geom.out_h, geom.out_w, sks.cout());
  detail::Staged dx(0, input.data(), input.size() * sizeof(T));
  detail::Staged dy(1, out.size() * sizeof(T));
  const segconv_geometry g = geom.c();
  throw_on(segconv_transpose_conv_fused(dx.get(), dtype_of<T>::value, 1, input.height(),
                                        input.channels(), &sks.desc, sks.panels->get(), &g,
                                        nullptr, SEGCONV_EPI_NONE, SEGCONV_MATH_AUTO, dy.get(),
                                        dtype_of<T>::value, nullptr));
  dy.to_host(out.data(), out.size() * sizeof(T));
  return out;
}

// reference fused_tconv.hpp:85-92
template <typename T>
Tensor<T> transpose_conv_fused(const Tensor<T>& input, const Kernel<T>& k, int p) {
  const TConvGeometry geom = tconv_geometry(input.height(), k.kh(), k.kw(), p);
  if (input.height() != input.width())
    throw ContractError("transpose conv expects a square input");
  return transpose_conv_fused(input, segregate(k, p), geom);
}

// reference fused_tconv.hpp:101-147: the GPU grid replaces the cout-slice
// threads; `workers` is validated as in the reference and the result is
// identical to transpose_conv_fused.
template <typename T>
Tensor<T> transpose_conv_fused_parallel(const Tensor<T>& input, const SubKernelSet<T>& sks,
                                        const TConvGeometry& geom, int workers) {
  if (workers < 1) throw ContractError("worker count must be >= 1");
  return transpose_conv_fused(input, sks, geom);
}

// reference reference_ops.hpp:86-108
template <typename T>
Tensor<T> conv2d_valid(const Tensor<T>& src, const Kernel<T>& k) {
  if (k.spatially_empty()) throw ShapeError("conv2d_valid needs a non-empty kernel");
  if (src.channels() != k.cin()) throw ContractError("channel mismatch");
  const int oh = src.height() - k.kh() + 1, ow = src.width() - k.kw() + 1;
  if (oh < 1 || ow < 1) throw ShapeError("kernel does not fit input");
  Tensor<T> out(oh, ow, k.cout());
  detail::Staged ds(0, src.data(), src.size() * sizeof(T)), dk(2, k.data(), k.size() * sizeof(T));
  detail::Staged dy(1, out.size() * sizeof(T));
  throw_on(segconv_conv2d_valid(ds.get(), dtype_of<T>::value, 1, src.height(), src.width(),
                                src.channels(), dk.get(), k.kh(), k.kw(), k.cout(), nullptr,
                                SEGCONV_EPI_NONE, dy.get(), nullptr));
  dy.to_host(out.data(), out.size() * sizeof(T));
  return out;
}

// reference reference_ops.hpp:116-133
template <typename T>
Tensor<T> transpose_conv_naive(const Tensor<T>& input, const Kernel<T>& k, int p) {
  if (input.channels() != k.cin()) throw ContractError("channel mismatch");
  const TConvGeometry geom = tconv_geometry(input.height(), k.kh(), k.kw(), p);
  if (input.height() != input.width())
    throw ContractError("transpose conv expects a square input");
  Tensor<T> out(geom.out_h, geom.out_w, k.cout());
  const size_t ws = segconv_naive_workspace_bytes(dtype_of<T>::value, 1, input.height(),
                                                  input.channels(), p);
  detail::Staged dx(0, input.data(), input.size() * sizeof(T)), dk(2, k.data(), k.size() * sizeof(T));
  detail::Staged dw(3, ws), dy(1, out.size() * sizeof(T));
  throw_on(segconv_transpose_conv_naive(dx.get(), dtype_of<T>::value, 1, input.height(),
                                        input.channels(), dk.get(), k.kh(), k.kw(), k.cout(), p,
                                        dw.get(), ws, nullptr, SEGCONV_EPI_NONE, dy.get(),
                                        nullptr));
  dy.to_host(out.data(), out.size() * sizeof(T));
  return out;
}

// ------------------------------------------------------------- SGC1 files
// reference tensor_io.hpp:46-103
enum class Precision { f32 = 0, f64 = 1 };
template <typename T>
inline constexpr Precision precision_of = std::is_same_v<T, double> ? Precision::f64 : Precision::f32;

struct TensorFileInfo {
  int height = 0, width = 0, channels = 0;
  Precision precision = Precision::f32;
};

inline TensorFileInfo peek_tensor_file(const std::string& path) {
  segconv_tensor_file_info i;
  throw_on(segconv_peek_tensor_file(path.c_str(), &i));
  return TensorFileInfo{i.height, i.width, i.channels, (Precision)i.precision};
}

template <typename T>
Tensor<T> load_tensor(const std::string& path) {
  const TensorFileInfo info = peek_tensor_file(path);
  Tensor<T> t(info.height, info.width, info.channels);
  throw_on(segconv_load_tensor(path.c_str(), dtype_of<T>::value, t.data(), t.size() * sizeof(T)));
  return t;
}

template <typename T>
void save_tensor(const Tensor<T>& t, const std::string& path) {
  throw_on(segconv_save_tensor(path.c_str(), t.data(), t.height(), t.width(), t.channels(),
                               dtype_of<T>::value));
}

// ------------------------------------------------------------- training layer
namespace net {

// reference netdemo/layers.hpp:23-29
template <typename T>
struct ParamBlock {
  T* values = nullptr;
  T* grads = nullptr;
  std::size_t size = 0;
};

// reference netdemo/layers.hpp:84-137 (net::ConvValid<T>): conv2d_valid forward,
// backward on the GPU (segconv_conv2d_valid_backward), host-side values/grads.
template <typename T>
class ConvValid {
 public:
  explicit ConvValid(Kernel<T> k, segconv_math math = SEGCONV_MATH_EXACT)
      : kernel_(std::move(k)), grad_(kernel_.kh(), kernel_.kw(), kernel_.cin(), kernel_.cout()), math_(math) {}
  const char* name() const { return "conv_valid"; }
  Tensor<T> forward(const Tensor<T>& in) {
    input_ = in;
    has_input_ = true;
    return conv2d_valid(in, kernel_);
  }
  Tensor<T> backward(const Tensor<T>& g) {
    if (!has_input_) throw StateError(std::string(name()) + ": backward called before forward");
    Tensor<T> gin(input_.height(), input_.width(), input_.channels());
    detail::Staged dx(0, input_.data(), input_.size() * sizeof(T)), dg(4, g.data(), g.size() * sizeof(T));
    detail::Staged dk(2, kernel_.data(), kernel_.size() * sizeof(T));
    detail::Staged dgk(5, grad_.data(), grad_.size() * sizeof(T)), dgx(1, gin.size() * sizeof(T));
    throw_on(segconv_conv2d_valid_backward(dx.get(), dg.get(), dtype_of<T>::value, 1, input_.height(),
                                           input_.width(), input_.channels(), dk.get(), kernel_.kh(),
                                           kernel_.kw(), kernel_.cout(), math_, dgx.get(), dgk.get(), 1, nullptr));
    dgx.to_host(gin.data(), gin.size() * sizeof(T));
    dgk.to_host(grad_.data(), grad_.size() * sizeof(T));
    return gin;
  }
  std::vector<ParamBlock<T>> params() { return {{kernel_.data(), grad_.data(), kernel_.size()}}; }
  const Kernel<T>& kernel() const { return kernel_; }

 private:
  Kernel<T> kernel_;
  Kernel<T> grad_;
  segconv_math math_;
  Tensor<T> input_;
  bool has_input_ = false;
};

// reference netdemo/layers.hpp:150-230 (net::FusedTConv<T>): forward runs the
// segregated GPU kernels, backward the GPU backward pass
// (segconv_transpose_conv_fused_backward); values and gradients live on the
// host as in the reference, so an optimizer written against params() works
// unchanged.  Default math EXACT: bit-identical to the reference layer.
template <typename T>
class FusedTConv {
 public:
  FusedTConv(Kernel<T> k, int p, segconv_math math = SEGCONV_MATH_EXACT)
      : kernel_(std::move(k)), grad_(kernel_.kh(), kernel_.kw(), kernel_.cin(), kernel_.cout()), p_(p),
        math_(math), sks_(segregate(kernel_, p, fwd_math(math))) {}

  const char* name() const { return "fused_tconv"; }

  Tensor<T> forward(const Tensor<T>& in) {
    if (in.height() != in.width())
      throw ContractError("fused_tconv expects a square input, got " + std::to_string(in.height()) + "x" +
                          std::to_string(in.width()));
    geom_ = tconv_geometry(in.height(), kernel_.kh(), kernel_.kw(), p_);
    input_ = in;
    has_input_ = true;
    return transpose_conv_fused(in, sks_, geom_);
  }

  Tensor<T> backward(const Tensor<T>& g) {
    if (!has_input_) throw StateError(std::string(name()) + ": backward called before forward");
    if (g.height() != geom_.out_h || g.width() != geom_.out_w || g.channels() != kernel_.cout())
      throw ContractError("fused_tconv: output gradient shape mismatch");
    Tensor<T> gin(input_.height(), input_.width(), input_.channels());
    detail::Staged dx(0, input_.data(), input_.size() * sizeof(T)), dg(4, g.data(), g.size() * sizeof(T));
    detail::Staged dk(2, kernel_.data(), kernel_.size() * sizeof(T));
    detail::Staged dgk(5, grad_.data(), grad_.size() * sizeof(T)), dgx(1, gin.size() * sizeof(T));
    throw_on(segconv_transpose_conv_fused_backward(
        dx.get(), dg.get(), dtype_of<T>::value, 1, input_.height(), input_.channels(), dk.get(), kernel_.kh(),
        kernel_.kw(), kernel_.cout(), p_, math_, dgx.get(), dgk.get(), /*accumulate=*/1, nullptr));
    dgx.to_host(gin.data(), gin.size() * sizeof(T));
    dgk.to_host(grad_.data(), grad_.size() * sizeof(T));
    return gin;
  }

  std::vector<ParamBlock<T>> params() { return {{kernel_.data(), grad_.data(), kernel_.size()}}; }
  void on_params_updated() { sks_ = segregate(kernel_, p_, fwd_math(math_)); }
  const Kernel<T>& kernel() const { return kernel_; }
  int padding() const { return p_; }

 private:
  static segconv_math fwd_math(segconv_math m) {
    return m == SEGCONV_MATH_EXACT ? SEGCONV_MATH_EXACT : SEGCONV_MATH_AUTO;
  }
  Kernel<T> kernel_;
  Kernel<T> grad_;
  int p_;
  segconv_math math_;
  SubKernelSet<T> sks_;
  TConvGeometry geom_{};
  Tensor<T> input_;
  bool has_input_ = false;
};

}  // namespace net

// reference tensor.hpp:263-286
template <typename T>
bool tensors_equal_exact(const Tensor<T>& a, const Tensor<T>& b) {
  if (!a.same_shape(b)) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a.data()[i] != b.data()[i]) return false;
  return true;
}
template <typename T>
bool tensors_equal_approx(const Tensor<T>& a, const Tensor<T>& b, T rel_tol) {
  if (!a.same_shape(b)) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    const T s = std::max({std::abs(a.data()[i]), std::abs(b.data()[i]), T(1)});
    if (std::abs(a.data()[i] - b.data()[i]) > rel_tol * s) return false;
  }
  return true;
}

}  // namespace segconv
