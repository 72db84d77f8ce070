// test_host_api.cpp -- exercises the drop-in C++ API (include/segconv_b200.hpp)
// the way the reference's own tests exercise proj/include: the frozen worked
// example, an independent scatter oracle on integer data (exact), the
// parallel variant, and the contract errors.  Exit code = number of failures.
#include <cstdio>
#include <random>

#include "segconv_b200.hpp"

using segconv::Kernel;
using segconv::Tensor;

static int failures = 0;
#define CHECK(cond, what)                                   \
  do {                                                      \
    if (!(cond)) {                                          \
      std::printf("FAIL %s\n", what);                       \
      ++failures;                                           \
    } else {                                                \
      std::printf("PASS %s\n", what);                       \
    }                                                       \
  } while (0)

// Scatter formulation (reference proj/tests/test_reference_ops.cpp:23-39 idea,
// written here from the definition): out(2i+p-u, 2j+p-v) += in(i,j,ch)*k(u,v,ch,f).
static std::vector<double> scatter(const Tensor<float>& in, const Kernel<float>& k, int p, int oh,
                                   int ow) {
  std::vector<double> out((size_t)oh * ow * k.cout(), 0.0);
  for (int i = 0; i < in.height(); ++i)
    for (int j = 0; j < in.width(); ++j)
      for (int u = 0; u < k.kh(); ++u)
        for (int v = 0; v < k.kw(); ++v) {
          const int y = 2 * i + p - u, x = 2 * j + p - v;
          if (y < 0 || y >= oh || x < 0 || x >= ow) continue;
          for (int ch = 0; ch < in.channels(); ++ch)
            for (int f = 0; f < k.cout(); ++f)
              out[((size_t)y * ow + x) * k.cout() + f] += (double)in(i, j, ch) * k(u, v, ch, f);
        }
  return out;
}

int main() {
  // frozen worked example: 2x2 [1,2,3,4], 3x3 ones, P=2 (test_reference_ops.cpp:96-112)
  {
    const auto in = Tensor<float>::from_data(2, 2, 1, {1, 2, 3, 4});
    const auto k = Kernel<float>::from_data(3, 3, 1, 1, std::vector<float>(9, 1.0f));
    const float want[5][5] = {{1, 1, 3, 2, 2}, {1, 1, 3, 2, 2}, {4, 4, 10, 6, 6},
                              {3, 3, 7, 4, 4}, {3, 3, 7, 4, 4}};
    const auto a = segconv::transpose_conv_naive(in, k, 2);
    const auto b = segconv::transpose_conv_fused(in, k, 2);
    bool ok = a.height() == 5 && b.height() == 5;
    for (int y = 0; ok && y < 5; ++y)
      for (int x = 0; x < 5; ++x) ok = ok && a(y, x, 0) == want[y][x] && b(y, x, 0) == want[y][x];
    CHECK(ok, "frozen worked example (naive and fused)");
  }
  // integer fuzz vs the scatter oracle, every math mode the API picks
  {
    std::mt19937 rng(20240911);
    std::uniform_int_distribution<int> d(-8, 8);
    int bad = 0, n_cases = 0;
    for (int t = 0; t < 60; ++t) {
      const int n = 1 + rng() % 9, p = rng() % 4;
      const int cap = std::min(7, 2 * n - 1 + 2 * p);
      const int kk = 1 + rng() % cap;
      const int cin = (t % 3 == 0) ? 16 * (1 + rng() % 3) : 1 + rng() % 4;
      const int cout = 1 + rng() % 40;
      Tensor<float> in(n, n, cin);
      for (size_t i = 0; i < in.size(); ++i) in.data()[i] = (float)d(rng);
      Kernel<float> k(kk, kk, cin, cout);
      for (size_t i = 0; i < k.size(); ++i) k.data()[i] = (float)d(rng);
      const auto y = segconv::transpose_conv_fused(in, k, p);
      const auto want = scatter(in, k, p, y.height(), y.width());
      for (size_t i = 0; i < want.size(); ++i)
        if ((double)y.data()[i] != want[i]) {
          ++bad;
          break;
        }
      ++n_cases;
    }
    std::printf("int fuzz: %d/%d cases exact\n", n_cases - bad, n_cases);
    CHECK(bad == 0, "integer fuzz == scatter oracle, exact");
  }
  // parallel variant == sequential; workers validated
  {
    std::mt19937 rng(1001);
    std::uniform_real_distribution<float> d(-1, 1);
    Tensor<float> in(9, 9, 2);
    for (size_t i = 0; i < in.size(); ++i) in.data()[i] = d(rng);
    Kernel<float> k(3, 3, 2, 37);
    for (size_t i = 0; i < k.size(); ++i) k.data()[i] = d(rng);
    const auto g = segconv::tconv_geometry(9, 3, 3, 1);
    const auto sks = segconv::segregate(k, 1);
    const auto seq = segconv::transpose_conv_fused(in, sks, g);
    bool ok = true;
    for (int w : {1, 2, 3, 4, 9})
      ok = ok && segconv::tensors_equal_exact(segconv::transpose_conv_fused_parallel(in, sks, g, w), seq);
    CHECK(ok, "fused_parallel == fused for workers 1,2,3,4,9");
    bool threw = false;
    try {
      segconv::transpose_conv_fused_parallel(in, sks, g, 0);
    } catch (const segconv::ContractError&) {
      threw = true;
    }
    CHECK(threw, "workers = 0 -> ContractError");
  }
  // contract and shape errors (test_reference_ops.cpp:151-160, test_fused.cpp:117-138)
  {
    bool c1 = false, c2 = false, c3 = false, c4 = false;
    try {
      segconv::transpose_conv_naive(Tensor<float>(2, 3, 1), Kernel<float>(3, 3, 1, 1), 1);
    } catch (const segconv::ContractError&) {
      c1 = true;
    }
    try {
      segconv::transpose_conv_naive(Tensor<float>(4, 4, 2), Kernel<float>(3, 3, 1, 1), 1);
    } catch (const segconv::ContractError&) {
      c2 = true;
    }
    try {
      segconv::transpose_conv_naive(Tensor<float>(4, 4, 2), Kernel<float>(9, 9, 2, 1), 0);
    } catch (const segconv::ShapeError&) {
      c3 = true;
    }
    try {
      const auto k = Kernel<float>::from_data(4, 4, 2, 2, std::vector<float>(64, 1.0f));
      segconv::transpose_conv_fused(Tensor<float>(6, 6, 2), segconv::segregate(k, 1),
                                    segconv::tconv_geometry(6, 4, 4, 2));
    } catch (const segconv::ContractError&) {
      c4 = true;
    }
    CHECK(c1 && c2 && c3 && c4, "rect / channel / extent / parity errors");
  }
  // SGC1 container (reference tests/test_io.cpp:44-127)
  {
    const std::string path = "/tmp/segconv_b200_test_host_api.sgc";
    std::mt19937 rng(44);
    std::uniform_real_distribution<double> d(-1, 1);
    Tensor<double> t(5, 4, 3);
    for (size_t i = 0; i < t.size(); ++i) t.data()[i] = d(rng);
    segconv::save_tensor(t, path);
    const auto info = segconv::peek_tensor_file(path);
    CHECK(info.height == 5 && info.width == 4 && info.channels == 3 &&
              info.precision == segconv::Precision::f64,
          "SGC1 header round trip");
    CHECK(segconv::tensors_equal_exact(segconv::load_tensor<double>(path), t), "SGC1 data round trip");
    bool c1 = false, c2 = false;
    try {
      segconv::load_tensor<float>(path);
    } catch (const segconv::ContractError&) {
      c1 = true;
    }
    std::FILE* f = std::fopen(path.c_str(), "wb");
    std::fwrite("SGC1xxxx", 1, 8, f);
    std::fclose(f);
    try {
      segconv::peek_tensor_file(path);
    } catch (const segconv::ParseError& e) {
      c2 = e.byte_offset == 8;
    }
    CHECK(c1 && c2, "SGC1 precision mismatch / short header errors");
    std::remove(path.c_str());
  }
  // trainable layer: forward + backward == scatter-form gradients on integer data
  {
    std::mt19937 rng(137);
    std::uniform_int_distribution<int> d(-3, 3);
    const int n = 5, cin = 3, cout = 2, kk = 4, p = 2;
    Tensor<double> in(n, n, cin);
    for (size_t i = 0; i < in.size(); ++i) in.data()[i] = d(rng);
    Kernel<double> k(kk, kk, cin, cout);
    for (size_t i = 0; i < k.size(); ++i) k.data()[i] = d(rng);
    segconv::net::FusedTConv<double> layer(k, p);
    bool state = false;
    try {
      layer.backward(Tensor<double>(8, 8, cout));
    } catch (const segconv::StateError&) {
      state = true;
    }
    CHECK(state, "layer backward before forward -> StateError");
    const auto y = layer.forward(in);
    Tensor<double> g(y.height(), y.width(), cout);
    for (size_t i = 0; i < g.size(); ++i) g.data()[i] = d(rng);
    const auto gin = layer.backward(g);
    const auto gin2 = layer.backward(g);  // tap gradients accumulate across calls
    bool ok = segconv::tensors_equal_exact(gin, gin2);
    const int oh = y.height(), ow = y.width();
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int ch = 0; ch < cin; ++ch) {
          double want = 0;
          for (int u = 0; u < kk; ++u)
            for (int v = 0; v < kk; ++v) {
              const int yy = 2 * i + p - u, xx = 2 * j + p - v;
              if (yy < 0 || yy >= oh || xx < 0 || xx >= ow) continue;
              for (int f = 0; f < cout; ++f) want += k(u, v, ch, f) * g(yy, xx, f);
            }
          ok = ok && gin(i, j, ch) == want;
        }
    auto blocks = layer.params();
    for (int u = 0; u < kk; ++u)
      for (int v = 0; v < kk; ++v)
        for (int ch = 0; ch < cin; ++ch)
          for (int f = 0; f < cout; ++f) {
            double want = 0;
            for (int i = 0; i < n; ++i)
              for (int j = 0; j < n; ++j) {
                const int yy = 2 * i + p - u, xx = 2 * j + p - v;
                if (yy < 0 || yy >= oh || xx < 0 || xx >= ow) continue;
                want += in(i, j, ch) * g(yy, xx, f);
              }
            ok = ok && blocks[0].grads[(((size_t)u * kk + v) * cin + ch) * cout + f] == 2 * want;
          }
    CHECK(ok && blocks.size() == 1 && blocks[0].size == k.size(), "layer gradients == scatter form, exact");
  }
  // ConvValid layer (reference layers.hpp:84-137): gradients on integer data, exact
  {
    std::mt19937 rng(98);
    std::uniform_int_distribution<int> d(-3, 3);
    const int h = 7, w = 6, cin = 2, cout = 3, kh = 3, kw = 2;
    Tensor<double> in(h, w, cin);
    for (size_t i = 0; i < in.size(); ++i) in.data()[i] = d(rng);
    Kernel<double> k(kh, kw, cin, cout);
    for (size_t i = 0; i < k.size(); ++i) k.data()[i] = d(rng);
    segconv::net::ConvValid<double> layer(k);
    const auto y = layer.forward(in);
    Tensor<double> g(y.height(), y.width(), cout);
    for (size_t i = 0; i < g.size(); ++i) g.data()[i] = d(rng);
    const auto gin = layer.backward(g);
    bool ok = true;
    for (int a = 0; a < h; ++a)
      for (int c = 0; c < w; ++c)
        for (int ch = 0; ch < cin; ++ch) {
          double want = 0;
          for (int u = 0; u < kh; ++u)
            for (int v = 0; v < kw; ++v) {
              const int yy = a - u, xx = c - v;
              if (yy < 0 || yy >= y.height() || xx < 0 || xx >= y.width()) continue;
              for (int f = 0; f < cout; ++f) want += k(u, v, ch, f) * g(yy, xx, f);
            }
          ok = ok && gin(a, c, ch) == want;
        }
    auto blocks = layer.params();
    for (int u = 0; u < kh; ++u)
      for (int v = 0; v < kw; ++v)
        for (int ch = 0; ch < cin; ++ch)
          for (int f = 0; f < cout; ++f) {
            double want = 0;
            for (int yy = 0; yy < y.height(); ++yy)
              for (int xx = 0; xx < y.width(); ++xx) want += in(yy + u, xx + v, ch) * g(yy, xx, f);
            ok = ok && blocks[0].grads[(((size_t)u * kw + v) * cin + ch) * cout + f] == want;
          }
    CHECK(ok, "ConvValid layer gradients == direct sums, exact");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
