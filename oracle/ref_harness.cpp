// ref_harness.cpp -- TEST INFRASTRUCTURE. A thin extern "C" shim over the
// UNMODIFIED reference headers (/root/reference/proj/include, included in
// place, never copied) so Python tests and bench.py can call the reference's
// own CPU implementation.  Built by oracle/Makefile into oracle/_ref/.
//
// Used for: (1) pinning oracle/segconv_oracle.c against the real reference,
// (2) generating tests/golden fixtures, (3) the CPU baseline
// (cpu_baseline.kind = "reference") and `bench.py --impl reference`.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "segconv/analysis.hpp"
#include "segconv/fused_tconv.hpp"
#include "segconv/geometry.hpp"
#include "segconv/netdemo/layers.hpp"
#include "segconv/reference_ops.hpp"
#include "segconv/segregation.hpp"
#include "segconv/tensor.hpp"
#include "segconv/tensor_io.hpp"
#include "segconv/verify.hpp"

namespace {

thread_local std::string g_err;
thread_local size_t g_offset = 0;

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const segconv::ParseError& e) {
    g_err = e.what();
    g_offset = e.byte_offset;
    return 6;
  } catch (const segconv::IoError& e) {
    g_err = e.what();
    return 5;
  } catch (const segconv::ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const segconv::ContractError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

template <typename T>
segconv::Tensor<T> image(const T* x, int n, int cin) {
  return segconv::Tensor<T>::from_data(n, n, cin, std::vector<T>(x, x + (size_t)n * n * cin));
}

template <typename T>
segconv::Kernel<T> kernel(const T* k, int kh, int kw, int cin, int cout) {
  return segconv::Kernel<T>::from_data(kh, kw, cin, cout,
                                       std::vector<T>(k, k + (size_t)kh * kw * cin * cout));
}

// variant: 0 fused(x, k, p), 1 naive, 2 fused_parallel(workers)
template <typename T>
int run_batch(int variant, const T* x, int batch, int n, int cin, const T* k, int kh, int kw,
              int cout, int p, int workers, T* out) {
  return guarded([&] {
    const auto kk = kernel(k, kh, kw, cin, cout);
    const auto geom = segconv::tconv_geometry(n, kh, kw, p);
    const auto sks = segconv::segregate(kk, p);
    const size_t isz = (size_t)n * n * cin;
    const size_t osz = (size_t)geom.out_h * geom.out_w * cout;
    for (int b = 0; b < batch; ++b) {
      const auto in = image(x + b * isz, n, cin);
      segconv::Tensor<T> y;
      if (variant == 0)
        y = segconv::transpose_conv_fused(in, kk, p);
      else if (variant == 1)
        y = segconv::transpose_conv_naive(in, kk, p);
      else
        y = segconv::transpose_conv_fused_parallel(in, sks, geom, workers);
      std::memcpy(out + b * osz, y.data(), osz * sizeof(T));
    }
  });
}


// Backward of the reference's trainable fused layer (netdemo/layers.hpp:171-211)
// over a batch: one FusedTConv, grads zeroed once (model.hpp:192), then per
// image forward + backward; gx per image, gk = the accumulated tap gradient.
template <typename T>
int run_backward(const T* x, int batch, int n, int cin, const T* k, int kh, int kw, int cout,
                 int p, const T* gy, T* gx, T* gk) {
  return guarded([&] {
    segconv::net::FusedTConv<T> layer(kernel(k, kh, kw, cin, cout), p);
    for (auto& blk : layer.params()) std::fill(blk.grads, blk.grads + blk.size, T(0));
    const auto geom = segconv::tconv_geometry(n, kh, kw, p);
    const size_t isz = (size_t)n * n * cin;
    const size_t osz = (size_t)geom.out_h * geom.out_w * cout;
    for (int b = 0; b < batch; ++b) {
      layer.forward(image(x + b * isz, n, cin));
      const auto g = segconv::Tensor<T>::from_data(geom.out_h, geom.out_w, cout,
                                                   std::vector<T>(gy + b * osz, gy + (b + 1) * osz));
      const auto gi = layer.backward(g);
      std::memcpy(gx + b * isz, gi.data(), isz * sizeof(T));
    }
    const auto blk = layer.params()[0];
    std::memcpy(gk, blk.grads, blk.size * sizeof(T));
  });
}

// net::ConvValid forward + backward per image (layers.hpp:84-122), grads zeroed once
template <typename T>
int run_conv_backward(const T* src, int batch, int h, int w, int cin, const T* k, int kh, int kw, int cout,
                      const T* gy, T* gx, T* gk) {
  return guarded([&] {
    segconv::net::ConvValid<T> layer(kernel(k, kh, kw, cin, cout));
    for (auto& blk : layer.params()) std::fill(blk.grads, blk.grads + blk.size, T(0));
    const int oh = h - kh + 1, ow = w - kw + 1;
    const size_t isz = (size_t)h * w * cin, osz = (size_t)oh * ow * cout;
    for (int b = 0; b < batch; ++b) {
      layer.forward(segconv::Tensor<T>::from_data(h, w, cin, std::vector<T>(src + b * isz, src + (b + 1) * isz)));
      const auto gi = layer.backward(
          segconv::Tensor<T>::from_data(oh, ow, cout, std::vector<T>(gy + b * osz, gy + (b + 1) * osz)));
      std::memcpy(gx + b * isz, gi.data(), isz * sizeof(T));
    }
    const auto blk = layer.params()[0];
    std::memcpy(gk, blk.grads, blk.size * sizeof(T));
  });
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
size_t ref_last_error_offset() { return g_offset; }

// SGC1 container through the reference's own tensor_io.hpp
int ref_save_tensor(const char* path, const void* data, int h, int w, int c, int f64) {
  return guarded([&] {
    if (f64)
      segconv::save_tensor(segconv::Tensor<double>::from_data(
                               h, w, c, std::vector<double>((const double*)data, (const double*)data + (size_t)h * w * c)),
                           path);
    else
      segconv::save_tensor(segconv::Tensor<float>::from_data(
                               h, w, c, std::vector<float>((const float*)data, (const float*)data + (size_t)h * w * c)),
                           path);
  });
}
// dims_out: h, w, c, precision; data copied into out (capacity in elements)
int ref_load_tensor(const char* path, int f64, void* out, size_t cap, int dims_out[4]) {
  return guarded([&] {
    const auto info = segconv::peek_tensor_file(path);
    dims_out[0] = info.height;
    dims_out[1] = info.width;
    dims_out[2] = info.channels;
    dims_out[3] = (int)info.precision;
    if (f64) {
      const auto t = segconv::load_tensor<double>(path);
      if (t.size() <= cap) std::memcpy(out, t.data(), t.size() * sizeof(double));
    } else {
      const auto t = segconv::load_tensor<float>(path);
      if (t.size() <= cap) std::memcpy(out, t.data(), t.size() * sizeof(float));
    }
  });
}

int ref_tconv_geometry(int n_in, int kh, int kw, int p, int out[11]) {
  return guarded([&] {
    const auto g = segconv::tconv_geometry(n_in, kh, kw, p);
    const int v[11] = {g.n_in,  g.kh,   g.kw,    g.p_orig,          g.p_fused,         g.up_h,
                       g.up_w,  g.out_h, g.out_w, (int)g.trim_extra_row, (int)g.trim_extra_col};
    std::memcpy(out, v, sizeof v);
  });
}

// panels: concatenated subs in class order r*2+c; dims/offs: 8 ints each.
int ref_segregate_f32(const float* k, int kh, int kw, int cin, int cout, int p, float* panels,
                      int dims[8], int offs[8]) {
  return guarded([&] {
    const auto sks = segconv::segregate(kernel(k, kh, kw, cin, cout), p);
    size_t w = 0;
    for (int q = 0; q < 4; ++q) {
      const auto& s = sks.subs[q];
      dims[2 * q] = s.kh();
      dims[2 * q + 1] = s.kw();
      offs[2 * q] = sks.class_input_offsets[q].first;
      offs[2 * q + 1] = sks.class_input_offsets[q].second;
      if (s.size()) std::memcpy(panels + w, s.data(), s.size() * sizeof(float));
      w += s.size();
    }
  });
}

int ref_tconv_fused_f32(const float* x, int batch, int n, int cin, const float* k, int kh, int kw,
                        int cout, int p, float* out) {
  return run_batch<float>(0, x, batch, n, cin, k, kh, kw, cout, p, 1, out);
}
int ref_tconv_naive_f32(const float* x, int batch, int n, int cin, const float* k, int kh, int kw,
                        int cout, int p, float* out) {
  return run_batch<float>(1, x, batch, n, cin, k, kh, kw, cout, p, 1, out);
}
int ref_tconv_fused_parallel_f32(const float* x, int batch, int n, int cin, const float* k,
                                 int kh, int kw, int cout, int p, int workers, float* out) {
  return run_batch<float>(2, x, batch, n, cin, k, kh, kw, cout, p, workers, out);
}
int ref_tconv_fused_f64(const double* x, int batch, int n, int cin, const double* k, int kh,
                        int kw, int cout, int p, double* out) {
  return run_batch<double>(0, x, batch, n, cin, k, kh, kw, cout, p, 1, out);
}
int ref_tconv_naive_f64(const double* x, int batch, int n, int cin, const double* k, int kh,
                        int kw, int cout, int p, double* out) {
  return run_batch<double>(1, x, batch, n, cin, k, kh, kw, cout, p, 1, out);
}

// out: naive mults, naive adds, fused mults, fused adds
int ref_count_ops(int n, int cin, int cout, int kh, int kw, int p, uint64_t out[4]) {
  return guarded([&] {
    const segconv::LayerShape s{n, cin, cout, kh, kw, p};
    const auto a = segconv::count_ops_naive(s);
    const auto b = segconv::count_ops_fused(s);
    out[0] = a.mults;
    out[1] = a.adds;
    out[2] = b.mults;
    out[3] = b.adds;
  });
}

// The reference fuzz, verbatim through its API: returns cases_run, failures,
// first failing case index (or -1).
int ref_run_verify(int cases, uint64_t seed, int inject_fault_case, int out[3]) {
  return guarded([&] {
    segconv::VerifyOptions opt;
    opt.cases = cases;
    opt.seed = seed;
    opt.inject_fault_case = inject_fault_case;
    const auto r = segconv::run_verify(opt);
    out[0] = r.cases_run;
    out[1] = r.failures;
    out[2] = r.first_failure ? r.first_failure->case_index : -1;
  });
}

// Replays run_verify's case generator (proj/include/segconv/verify.hpp:66-93,
// same engine and distributions, default ranges) and returns case `want`:
// dims[5] = n, k, p, cin, cout; x/kernel values written to x_out/k_out
// (caller provides >= 16*16*4 and 7*7*4*4 floats).  The reference output is
// produced by the reference's transpose_conv_naive for the same case.
int ref_verify_case(uint64_t seed, int want, int dims[5], float* x_out, float* k_out,
                    float* y_out) {
  return guarded([&] {
    const segconv::VerifyOptions opt;
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int> n_dist(opt.n_min, opt.n_max);
    std::uniform_int_distribution<int> p_dist(opt.p_min, opt.p_max);
    std::uniform_int_distribution<int> c_dist(opt.c_min, opt.c_max);
    std::uniform_int_distribution<int> value_dist(-8, 8);
    for (int case_i = 0; case_i <= want; ++case_i) {
      const int n = n_dist(rng);
      const int p = p_dist(rng);
      const int k_cap = std::min(opt.k_max, 2 * n - 1 + 2 * p);
      std::uniform_int_distribution<int> k_dist(std::min(opt.k_min, k_cap), k_cap);
      const int k = k_dist(rng);
      const int cin = c_dist(rng);
      const int cout = c_dist(rng);
      std::vector<float> xd((size_t)n * n * cin);
      for (float& v : xd) v = (float)value_dist(rng);
      std::vector<float> kd((size_t)k * k * cin * cout);
      for (float& v : kd) v = (float)value_dist(rng);
      if (case_i == want) {
        dims[0] = n;
        dims[1] = k;
        dims[2] = p;
        dims[3] = cin;
        dims[4] = cout;
        std::memcpy(x_out, xd.data(), xd.size() * sizeof(float));
        std::memcpy(k_out, kd.data(), kd.size() * sizeof(float));
        const auto in = segconv::Tensor<float>::from_data(n, n, cin, xd);
        const auto kk = segconv::Kernel<float>::from_data(k, k, cin, cout, kd);
        const auto y = segconv::transpose_conv_naive(in, kk, p);
        std::memcpy(y_out, y.data(), y.size() * sizeof(float));
      }
    }
  });
}

// CPU baseline timing of the reference's own segregated path over a batch.
// mode 0: loop images through transpose_conv_fused_parallel(workers) (the
//         reference's own threading: contiguous cout slices, capped at cout);
// mode 1: harness-level batch threading -- `workers` threads each run the
//         reference's sequential transpose_conv_fused on whole images
//         (workers = 1: the sequential op alone);
// mode 2: as mode 1 with the conventional transpose_conv_naive
//         (reference_ops.hpp:116-133: upsample + pad + valid conv).
// Segregation happens outside the timed region (proj/include/segconv/bench.hpp:83).
// Returns wall seconds in *seconds.
int ref_time_fused_batch_f32(int mode, const float* x, int batch, int n, int cin, const float* k,
                             int kh, int kw, int cout, int p, int workers, float* out,
                             double* seconds) {
  return guarded([&] {
    const auto kk = kernel(k, kh, kw, cin, cout);
    const auto geom = segconv::tconv_geometry(n, kh, kw, p);
    const auto sks = segconv::segregate(kk, p);
    const size_t isz = (size_t)n * n * cin;
    const size_t osz = (size_t)geom.out_h * geom.out_w * cout;
    std::vector<segconv::Tensor<float>> ins;
    ins.reserve(batch);
    for (int b = 0; b < batch; ++b) ins.push_back(image(x + b * isz, n, cin));
    const auto t0 = std::chrono::steady_clock::now();
    if (mode == 0) {
      for (int b = 0; b < batch; ++b) {
        const auto y = segconv::transpose_conv_fused_parallel(ins[b], sks, geom, workers);
        std::memcpy(out + b * osz, y.data(), osz * sizeof(float));
      }
    } else {
      std::atomic<int> next{0};
      auto work = [&] {
        for (int b = next++; b < batch; b = next++) {
          const auto y = mode == 2 ? segconv::transpose_conv_naive(ins[b], kk, p)
                                   : segconv::transpose_conv_fused(ins[b], sks, geom);
          std::memcpy(out + b * osz, y.data(), osz * sizeof(float));
        }
      };
      std::vector<std::thread> pool;
      const int nt = std::max(1, std::min(workers, batch));
      for (int t = 0; t < nt; ++t) pool.emplace_back(work);
      for (auto& th : pool) th.join();
    }
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

// reference_ops.hpp:86-108 (conv2d_valid) over a batch of (h, w, cin) maps
int ref_conv2d_valid_f32(const float* src, int batch, int h, int w, int cin, const float* k, int kh, int kw,
                         int cout, float* out) {
  return guarded([&] {
    const auto kk = kernel(k, kh, kw, cin, cout);
    const size_t isz = (size_t)h * w * cin, osz = (size_t)(h - kh + 1) * (w - kw + 1) * cout;
    for (int b = 0; b < batch; ++b) {
      const auto in = segconv::Tensor<float>::from_data(h, w, cin,
                                                        std::vector<float>(src + b * isz, src + (b + 1) * isz));
      const auto y = segconv::conv2d_valid(in, kk);
      std::memcpy(out + b * osz, y.data(), osz * sizeof(float));
    }
  });
}

int ref_conv2d_valid_backward_f32(const float* src, int batch, int h, int w, int cin, const float* k, int kh,
                                  int kw, int cout, const float* gy, float* gx, float* gk) {
  return run_conv_backward<float>(src, batch, h, w, cin, k, kh, kw, cout, gy, gx, gk);
}
int ref_conv2d_valid_backward_f64(const double* src, int batch, int h, int w, int cin, const double* k, int kh,
                                  int kw, int cout, const double* gy, double* gx, double* gk) {
  return run_conv_backward<double>(src, batch, h, w, cin, k, kh, kw, cout, gy, gx, gk);
}

int ref_tconv_backward_f32(const float* x, int batch, int n, int cin, const float* k, int kh,
                           int kw, int cout, int p, const float* gy, float* gx, float* gk) {
  return run_backward<float>(x, batch, n, cin, k, kh, kw, cout, p, gy, gx, gk);
}
int ref_tconv_backward_f64(const double* x, int batch, int n, int cin, const double* k, int kh,
                           int kw, int cout, int p, const double* gy, double* gx, double* gk) {
  return run_backward<double>(x, batch, n, cin, k, kh, kw, cout, p, gy, gx, gk);
}

// CPU baseline timing of the reference backward: `workers` threads each own a
// FusedTConv and run forward + backward over a contiguous slice of the batch
// (the layer caches its input, so one layer cannot be shared across threads).
int ref_time_backward_f32(const float* x, int batch, int n, int cin, const float* k, int kh, int kw,
                          int cout, int p, const float* gy, int workers, float* gx, float* gk,
                          double* seconds) {
  return guarded([&] {
    const auto geom = segconv::tconv_geometry(n, kh, kw, p);
    const size_t isz = (size_t)n * n * cin;
    const size_t osz = (size_t)geom.out_h * geom.out_w * cout;
    const size_t ksz = (size_t)kh * kw * cin * cout;
    const int nt = std::max(1, std::min(workers, batch));
    std::vector<std::unique_ptr<segconv::net::FusedTConv<float>>> layers;
    for (int t = 0; t < nt; ++t) {
      layers.emplace_back(new segconv::net::FusedTConv<float>(kernel(k, kh, kw, cin, cout), p));
      for (auto& blk : layers.back()->params()) std::fill(blk.grads, blk.grads + blk.size, 0.0f);
    }
    std::vector<segconv::Tensor<float>> ins, gs;
    for (int b = 0; b < batch; ++b) {
      ins.push_back(image(x + b * isz, n, cin));
      gs.push_back(segconv::Tensor<float>::from_data(
          geom.out_h, geom.out_w, cout, std::vector<float>(gy + b * osz, gy + (b + 1) * osz)));
    }
    // the forward each backward needs (the layer caches its input) is run but not
    // timed: seconds = max over threads of that thread's backward time + the
    // final sum of the per-thread tap gradients
    std::vector<double> busy(nt, 0.0);
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        const int b0 = (int)((long long)batch * t / nt), b1 = (int)((long long)batch * (t + 1) / nt);
        for (int b = b0; b < b1; ++b) {
          layers[t]->forward(ins[b]);
          const auto a = std::chrono::steady_clock::now();
          const auto gi = layers[t]->backward(gs[b]);
          busy[t] += std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
          std::memcpy(gx + b * isz, gi.data(), isz * sizeof(float));
        }
      });
    for (auto& th : pool) th.join();
    const auto t0 = std::chrono::steady_clock::now();
    std::memset(gk, 0, ksz * sizeof(float));
    for (int t = 0; t < nt; ++t) {
      const float* g = layers[t]->params()[0].grads;
      for (size_t e = 0; e < ksz; ++e) gk[e] += g[e];
    }
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = *std::max_element(busy.begin(), busy.end()) + std::chrono::duration<double>(t1 - t0).count();
  });
}

}  // extern "C"
