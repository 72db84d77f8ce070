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
#include <array>
#include <cmath>
#include <cstdint>
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

// Arithmetic of the value-semantics operators.  AUTO: the tensor-core kernels
// where the layer suits them (fp32 data: split-fp16, within 1e-5 of the
// reference).  Build with -DSEGCONV_B200_DEFAULT_MATH=SEGCONV_MATH_EXACT to get
// the reference's bit-for-bit results everywhere (its accumulation order, no
// FMA contraction), e.g. to run the reference's samples unchanged.
#ifndef SEGCONV_B200_DEFAULT_MATH
#define SEGCONV_B200_DEFAULT_MATH SEGCONV_MATH_AUTO
#endif

// ------------------------------------------------------------- allocation accounting
// reference tensor.hpp:22-55: Tensor / Kernel host storage allocated inside an
// active AllocScope is tallied into its AllocStats.  The device work of the
// operators allocates no host tensors, so a fused call records only its output
// (the reference's also records its padded input copy).
struct AllocStats {
  std::size_t total_bytes = 0;
  std::size_t peak_single = 0;
  std::size_t allocations = 0;
  void note(std::size_t bytes) {
    total_bytes += bytes;
    peak_single = std::max(peak_single, bytes);
    ++allocations;
  }
};

class AllocScope {
 public:
  explicit AllocScope(AllocStats& stats) : prev_(current_) { current_ = &stats; }
  ~AllocScope() { current_ = prev_; }
  AllocScope(const AllocScope&) = delete;
  AllocScope& operator=(const AllocScope&) = delete;
  static void note(std::size_t bytes) {
    if (current_ != nullptr) current_->note(bytes);
  }

 private:
  AllocStats* prev_;
  static inline thread_local AllocStats* current_ = nullptr;
};

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
    check_dims(h, w, c);
    data_.assign(size(), T(0));
    AllocScope::note(size() * sizeof(T));
  }
  static Tensor from_data(int h, int w, int c, std::vector<T> values) {
    check_dims(h, w, c);
    const std::size_t expect = (std::size_t)h * (std::size_t)w * (std::size_t)c;
    if (values.size() != expect)
      throw ContractError("tensor data length " + std::to_string(values.size()) + " does not match dims (" +
                          std::to_string(h) + "x" + std::to_string(w) + "x" + std::to_string(c) + ")");
    for (const T v : values)
      if (!std::isfinite(v)) throw ContractError("tensor data contains a non-finite element");
    Tensor t;
    t.h_ = h;
    t.w_ = w;
    t.c_ = c;
    t.data_ = std::move(values);
    AllocScope::note(t.size() * sizeof(T));
    return t;
  }
  Tensor(const Tensor& o) : h_(o.h_), w_(o.w_), c_(o.c_), data_(o.data_) {
    AllocScope::note(data_.size() * sizeof(T));
  }
  Tensor& operator=(const Tensor& o) {
    if (this != &o) {
      h_ = o.h_;
      w_ = o.w_;
      c_ = o.c_;
      data_ = o.data_;
      AllocScope::note(data_.size() * sizeof(T));
    }
    return *this;
  }
  Tensor(Tensor&&) noexcept = default;
  Tensor& operator=(Tensor&&) noexcept = default;

  int height() const { return h_; }
  int width() const { return w_; }
  int channels() const { return c_; }
  size_t size() const { return (size_t)h_ * w_ * c_; }
  bool empty() const { return data_.empty(); }
  size_t index(int i, int j, int ch) const { return ((size_t)i * w_ + j) * c_ + ch; }
  T operator()(int i, int j, int ch) const { return data_[index(i, j, ch)]; }
  T& operator()(int i, int j, int ch) { return data_[index(i, j, ch)]; }
  const T* pixel(int i, int j) const { return data_.data() + index(i, j, 0); }
  T* pixel(int i, int j) { return data_.data() + index(i, j, 0); }
  const T* data() const { return data_.data(); }
  T* data() { return data_.data(); }
  const std::vector<T>& storage() const { return data_; }
  bool same_shape(const Tensor& o) const { return h_ == o.h_ && w_ == o.w_ && c_ == o.c_; }

 private:
  static void check_dims(int h, int w, int c) {
    if (h < 1 || w < 1 || c < 1)
      throw ShapeError("tensor dims must be positive, got " + std::to_string(h) + "x" + std::to_string(w) + "x" +
                       std::to_string(c));
  }
  int h_ = 0, w_ = 0, c_ = 0;
  std::vector<T> data_;
};

// (kh, kw, cin, cout), cout innermost (reference tensor.hpp:152-217)
template <typename T>
class Kernel {
  static_assert(std::is_floating_point_v<T>, "Kernel requires float or double");

 public:
  Kernel() = default;
  // spatial dims may be zero: segregation produces legal empty sub-kernels
  Kernel(int kh, int kw, int cin, int cout) : kh_(kh), kw_(kw), cin_(cin), cout_(cout) {
    if (kh < 0 || kw < 0 || cin < 1 || cout < 1) throw ShapeError("bad kernel dims " + dims(kh, kw, cin, cout));
    data_.assign(size(), T(0));
    AllocScope::note(size() * sizeof(T));
  }
  static Kernel from_data(int kh, int kw, int cin, int cout, std::vector<T> values) {
    if (kh < 1 || kw < 1 || cin < 1 || cout < 1) throw ShapeError("bad kernel dims " + dims(kh, kw, cin, cout));
    const std::size_t expect = (std::size_t)kh * kw * cin * cout;
    if (values.size() != expect)
      throw ContractError("kernel data length " + std::to_string(values.size()) + " does not match dims " +
                          dims(kh, kw, cin, cout));
    for (const T v : values)
      if (!std::isfinite(v)) throw ContractError("kernel data contains a non-finite element");
    Kernel k;
    k.kh_ = kh;
    k.kw_ = kw;
    k.cin_ = cin;
    k.cout_ = cout;
    k.data_ = std::move(values);
    AllocScope::note(k.size() * sizeof(T));
    return k;
  }
  int kh() const { return kh_; }
  int kw() const { return kw_; }
  int cin() const { return cin_; }
  int cout() const { return cout_; }
  size_t size() const { return (size_t)kh_ * kw_ * cin_ * cout_; }
  bool spatially_empty() const { return kh_ == 0 || kw_ == 0; }
  size_t index(int u, int v, int ch, int f) const { return (((size_t)u * kw_ + v) * cin_ + ch) * cout_ + f; }
  T operator()(int u, int v, int ch, int f) const { return data_[index(u, v, ch, f)]; }
  T& operator()(int u, int v, int ch, int f) { return data_[index(u, v, ch, f)]; }
  // the cout values of tap (u, v, ch)
  const T* tap(int u, int v, int ch) const { return data_.data() + index(u, v, ch, 0); }
  const T* data() const { return data_.data(); }
  T* data() { return data_.data(); }

 private:
  static std::string dims(int kh, int kw, int cin, int cout) {
    return std::to_string(kh) + "x" + std::to_string(kw) + "x" + std::to_string(cin) + "x" + std::to_string(cout);
  }
  int kh_ = 0, kw_ = 0, cin_ = 0, cout_ = 0;
  std::vector<T> data_;
};

// ------------------------------------------------------------- op counts
// reference op_counts.hpp:9-41: multiply / add tallies; the counting hooks of
// the TallyT overloads below.  The device kernels do not count as they go: a
// TallyT overload adds the analytic totals of the call (the reference's
// dots(count, len) per output pixel summed over the pixels -- equal totals).
struct OpCounts {
  std::uint64_t mults = 0;
  std::uint64_t adds = 0;
  OpCounts& operator+=(const OpCounts& o) {
    mults += o.mults;
    adds += o.adds;
    return *this;
  }
  friend OpCounts operator+(OpCounts a, const OpCounts& b) { return a += b; }
  friend bool operator==(const OpCounts& a, const OpCounts& b) { return a.mults == b.mults && a.adds == b.adds; }
};
struct NoTally {
  static constexpr bool counting = false;
  void dots(std::uint64_t, std::uint64_t) {}
};
struct Tally {
  static constexpr bool counting = true;
  OpCounts counts;
  void dots(std::uint64_t count, std::uint64_t len) {
    counts.mults += count * len;
    if (len > 0) counts.adds += count * (len - 1);
  }
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
// reference segregation.hpp:91-101: sub-kernel sizes of an odd n x n kernel,
// largest class first.
inline std::array<std::pair<int, int>, 4> sub_kernel_dims(int n) {
  if (n < 1) throw ContractError("kernel size must be >= 1");
  if (n % 2 == 0) throw ContractError("sub_kernel_dims is defined for odd sizes only");
  const int hi = (n + 1) / 2, lo = n / 2;
  return {{{hi, hi}, {hi, lo}, {lo, hi}, {lo, lo}}};
}

// reference segregation.hpp:38-55.  `subs` / `class_input_offsets` are the
// reference's host-visible members (class q = r*2 + c); `desc` + `panels`
// are the device panels segconv_segregate wrote for the consumer kernel.
template <typename T>
struct SubKernelSet {
  std::array<Kernel<T>, 4> subs;
  std::array<std::pair<int, int>, 4> class_input_offsets;
  int source_kh = 0, source_kw = 0, p_orig_parity = 0;
  segconv_subkernels desc{};
  std::shared_ptr<DeviceBuffer> panels;
  const Kernel<T>& sub(int r, int c) const { return subs[r * 2 + c]; }
  std::pair<int, int> offset(int r, int c) const { return class_input_offsets[r * 2 + c]; }
  int cin() const { return desc.cin; }
  int cout() const { return desc.cout; }
};

// reference segregation.hpp:61-89.  The device panels come from one gather
// kernel (segconv_segregate); the host `subs` are the same taps,
// k[u0 + 2u][v0 + 2v][ch][f].  `math` picks the consumer kernel family.
template <typename T>
SubKernelSet<T> segregate(const Kernel<T>& k, int p_orig, segconv_math math = SEGCONV_B200_DEFAULT_MATH) {
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
  for (int q = 0; q < 4; ++q) {
    const int u0 = s.desc.u0[q], v0 = s.desc.v0[q], skh = s.desc.sub_kh[q], skw = s.desc.sub_kw[q];
    Kernel<T> sub(skh, skw, k.cin(), k.cout());
    for (int u = 0; u < skh; ++u)
      for (int v = 0; v < skw; ++v)
        for (int ch = 0; ch < k.cin(); ++ch)
          std::memcpy(&sub(u, v, ch, 0), k.tap(u0 + 2 * u, v0 + 2 * v, ch), k.cout() * sizeof(T));
    s.subs[q] = std::move(sub);
    s.class_input_offsets[q] = {s.desc.off_r[q], s.desc.off_c[q]};
  }
  return s;
}

// ------------------------------------------------------------- tensor ops
// reference tensor.hpp:224-259.  pad / crop are host copies (the device path
// never materialises them: the kernels predicate their halo loads);
// upsample2x runs the conventional path's device kernel (K5).
template <typename T>
Tensor<T> pad(const Tensor<T>& t, int p) {
  if (p < 0) throw ContractError("pad factor must be non-negative");
  Tensor<T> out(t.height() + 2 * p, t.width() + 2 * p, t.channels());
  const size_t row = (size_t)t.width() * t.channels() * sizeof(T);
  for (int i = 0; i < t.height(); ++i) std::memcpy(out.pixel(i + p, p), t.pixel(i, 0), row);
  return out;
}

template <typename T>
Tensor<T> crop(const Tensor<T>& t, int top, int left, int h, int w) {
  if (top < 0 || left < 0 || h < 1 || w < 1 || top + h > t.height() || left + w > t.width())
    throw ContractError("crop window out of range");
  Tensor<T> out(h, w, t.channels());
  const size_t row = (size_t)w * t.channels() * sizeof(T);
  for (int i = 0; i < h; ++i) std::memcpy(out.pixel(i, 0), t.pixel(top + i, left), row);
  return out;
}

template <typename T>
Tensor<T> upsample2x(const Tensor<T>& t) {
  Tensor<T> out(2 * t.height() - 1, 2 * t.width() - 1, t.channels());
  if (t.height() != t.width()) {  // the device kernel takes square maps (the operators' inputs)
    for (int i = 0; i < t.height(); ++i)
      for (int j = 0; j < t.width(); ++j)
        std::memcpy(out.pixel(2 * i, 2 * j), t.pixel(i, j), t.channels() * sizeof(T));
    return out;
  }
  detail::Staged dx(0, t.data(), t.size() * sizeof(T)), dy(1, out.size() * sizeof(T));
  throw_on(segconv_upsample2x_pad(dx.get(), dtype_of<T>::value, 1, t.height(), t.channels(), 0, dy.get(),
                                  nullptr));
  dy.to_host(out.data(), out.size() * sizeof(T));
  return out;
}

// ------------------------------------------------------------- operators
namespace detail {
// reference fused_tconv.hpp:17-35 (same messages; the C ABI checks again)
template <typename T>
void check_fused_args(const Tensor<T>& input, const SubKernelSet<T>& sks, const TConvGeometry& geom) {
  if (input.height() != geom.n_in || input.width() != geom.n_in)
    throw ContractError("input is " + std::to_string(input.height()) + "x" + std::to_string(input.width()) +
                        " but geometry was built for " + std::to_string(geom.n_in) + "x" +
                        std::to_string(geom.n_in));
  if (input.channels() != sks.cin())
    throw ContractError("channel mismatch: input has " + std::to_string(input.channels()) +
                        ", sub-kernels expect " + std::to_string(sks.cin()));
  if (sks.source_kh != geom.kh || sks.source_kw != geom.kw)
    throw ContractError("sub-kernel set was built from a " + std::to_string(sks.source_kh) + "x" +
                        std::to_string(sks.source_kw) + " kernel, geometry expects " + std::to_string(geom.kh) +
                        "x" + std::to_string(geom.kw));
  if (sks.p_orig_parity != (geom.p_orig & 1))
    throw ContractError("sub-kernel set was segregated for padding parity " + std::to_string(sks.p_orig_parity) +
                        ", geometry has p_orig " + std::to_string(geom.p_orig));
}
// the math of the conventional operators under SEGCONV_B200_DEFAULT_MATH
constexpr segconv_math conventional_math() {
  return SEGCONV_B200_DEFAULT_MATH == SEGCONV_MATH_EXACT || SEGCONV_B200_DEFAULT_MATH == SEGCONV_MATH_FFMA
             ? SEGCONV_B200_DEFAULT_MATH
             : SEGCONV_MATH_AUTO;
}
}  // namespace detail

// reference fused_tconv.hpp:69-82; the TallyT overload adds the call's
// multiply / add totals (reference fused_from_padded: dots(cout, taps * cin)
// per output pixel of each class)
template <typename T, typename TallyT>
Tensor<T> transpose_conv_fused(const Tensor<T>& input, const SubKernelSet<T>& sks, const TConvGeometry& geom,
                               TallyT& tally) {
  detail::check_fused_args(input, sks, geom);
  Tensor<T> out(geom.out_h, geom.out_w, sks.cout());
  detail::Staged dx(0, input.data(), input.size() * sizeof(T));
  detail::Staged dy(1, out.size() * sizeof(T));
  const segconv_geometry g = geom.c();
  throw_on(segconv_transpose_conv_fused(dx.get(), dtype_of<T>::value, 1, input.height(), input.channels(),
                                        &sks.desc, sks.panels->get(), &g, nullptr, SEGCONV_EPI_NONE,
                                        SEGCONV_MATH_AUTO, dy.get(), dtype_of<T>::value, nullptr));
  dy.to_host(out.data(), out.size() * sizeof(T));
  for (int q = 0; q < 4; ++q) {
    const int r = q >> 1, c = q & 1;
    const std::uint64_t pixels = (std::uint64_t)((geom.out_h - r + 1) / 2) * ((geom.out_w - c + 1) / 2);
    tally.dots(pixels * (std::uint64_t)sks.cout(),
               (std::uint64_t)sks.desc.sub_kh[q] * sks.desc.sub_kw[q] * sks.cin());
  }
  return out;
}

template <typename T>
Tensor<T> transpose_conv_fused(const Tensor<T>& input, const SubKernelSet<T>& sks, const TConvGeometry& geom) {
  NoTally t;
  return transpose_conv_fused(input, sks, geom, t);
}

// reference fused_tconv.hpp:85-92
template <typename T>
Tensor<T> transpose_conv_fused(const Tensor<T>& input, const Kernel<T>& k, int p) {
  const TConvGeometry geom = tconv_geometry(input.height(), k.kh(), k.kw(), p);
  if (input.height() != input.width())
    throw ContractError("transpose conv expects a square input, got " + std::to_string(input.height()) + "x" +
                        std::to_string(input.width()));
  return transpose_conv_fused(input, segregate(k, p), geom);
}

// reference fused_tconv.hpp:101-147: the GPU grid replaces the cout-slice
// threads; `workers` is validated as in the reference and the result is
// identical to transpose_conv_fused (as the reference's is for any count).
template <typename T>
Tensor<T> transpose_conv_fused_parallel(const Tensor<T>& input, const SubKernelSet<T>& sks,
                                        const TConvGeometry& geom, int workers) {
  if (workers < 1) throw ContractError("worker count must be >= 1");
  return transpose_conv_fused(input, sks, geom);
}

// reference reference_ops.hpp:86-108
template <typename T, typename TallyT>
Tensor<T> conv2d_valid(const Tensor<T>& src, const Kernel<T>& k, TallyT& tally) {
  if (k.spatially_empty()) throw ShapeError("conv2d_valid needs a non-empty kernel");
  if (src.channels() != k.cin())
    throw ContractError("channel mismatch: input has " + std::to_string(src.channels()) + ", kernel expects " +
                        std::to_string(k.cin()));
  const int oh = src.height() - k.kh() + 1, ow = src.width() - k.kw() + 1;
  if (oh < 1 || ow < 1) throw ShapeError("kernel does not fit input");
  Tensor<T> out(oh, ow, k.cout());
  detail::Staged ds(0, src.data(), src.size() * sizeof(T)), dk(2, k.data(), k.size() * sizeof(T));
  detail::Staged dy(1, out.size() * sizeof(T));
  throw_on(segconv_conv2d_valid(ds.get(), dtype_of<T>::value, 1, src.height(), src.width(), src.channels(),
                                dk.get(), k.kh(), k.kw(), k.cout(), nullptr, SEGCONV_EPI_NONE,
                                detail::conventional_math(), dy.get(), nullptr));
  dy.to_host(out.data(), out.size() * sizeof(T));
  tally.dots((std::uint64_t)oh * ow * k.cout(), (std::uint64_t)k.kh() * k.kw() * k.cin());
  return out;
}

template <typename T>
Tensor<T> conv2d_valid(const Tensor<T>& src, const Kernel<T>& k) {
  NoTally t;
  return conv2d_valid(src, k, t);
}

// reference reference_ops.hpp:116-133
template <typename T, typename TallyT>
Tensor<T> transpose_conv_naive(const Tensor<T>& input, const Kernel<T>& k, int p, TallyT& tally) {
  if (input.channels() != k.cin())
    throw ContractError("channel mismatch: input has " + std::to_string(input.channels()) + ", kernel expects " +
                        std::to_string(k.cin()));
  const TConvGeometry geom = tconv_geometry(input.height(), k.kh(), k.kw(), p);
  if (input.height() != input.width())
    throw ContractError("transpose conv expects a square input, got " + std::to_string(input.height()) + "x" +
                        std::to_string(input.width()));
  Tensor<T> out(geom.out_h, geom.out_w, k.cout());
  const size_t ws = segconv_naive_workspace_bytes(dtype_of<T>::value, 1, input.height(), input.channels(), p);
  detail::Staged dx(0, input.data(), input.size() * sizeof(T)), dk(2, k.data(), k.size() * sizeof(T));
  detail::Staged dw(3, ws), dy(1, out.size() * sizeof(T));
  throw_on(segconv_transpose_conv_naive(dx.get(), dtype_of<T>::value, 1, input.height(), input.channels(),
                                        dk.get(), k.kh(), k.kw(), k.cout(), p, dw.get(), ws, nullptr,
                                        SEGCONV_EPI_NONE, detail::conventional_math(), dy.get(), nullptr));
  dy.to_host(out.data(), out.size() * sizeof(T));
  tally.dots((std::uint64_t)geom.out_h * geom.out_w * k.cout(), (std::uint64_t)k.kh() * k.kw() * k.cin());
  return out;
}

template <typename T>
Tensor<T> transpose_conv_naive(const Tensor<T>& input, const Kernel<T>& k, int p) {
  NoTally t;
  return transpose_conv_naive(input, k, p, t);
}

// ------------------------------------------------------------- analysis
// reference analysis.hpp:14-77
struct LayerShape {
  int n_in = 0, cin = 0, cout = 0, kh = 0, kw = 0, p_orig = 0;
};
inline TConvGeometry geometry_of(const LayerShape& s) {
  if (s.cin < 1 || s.cout < 1)
    throw ShapeError("channel counts must be positive, got cin=" + std::to_string(s.cin) +
                     " cout=" + std::to_string(s.cout));
  return tconv_geometry(s.n_in, s.kh, s.kw, s.p_orig);
}
inline OpCounts count_ops_naive(const LayerShape& s) {
  uint64_t o[4];
  throw_on(segconv_count_ops(s.n_in, s.cin, s.cout, s.kh, s.kw, s.p_orig, o));
  return {o[0], o[1]};
}
inline OpCounts count_ops_fused(const LayerShape& s) {
  uint64_t o[4];
  throw_on(segconv_count_ops(s.n_in, s.cin, s.cout, s.kh, s.kw, s.p_orig, o));
  return {o[2], o[3]};
}
inline std::uint64_t memory_saved_bytes(const LayerShape& s, int elem_bytes) {
  const TConvGeometry g = geometry_of(s);
  const std::uint64_t up = (std::uint64_t)g.up_h * g.up_w;
  const std::uint64_t side = (std::uint64_t)s.n_in + 2 * g.p_fused;
  return (std::uint64_t)elem_bytes * (std::uint64_t)s.cin * (up - side * side);
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
