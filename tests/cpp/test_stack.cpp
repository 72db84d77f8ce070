// test_stack.cpp -- the C ABI's multi-GPU layer-stack driver (segconv_stack_*)
// from C++, on every visible GPU (1 on the test box): a three-layer fp32
// chain with bias + ReLU between layers and tanh at the end, checked against
// a double-precision scatter restatement of the reference semantics
// (out(2i+p-u, 2j+p-v) += in(i,j,ch) * k(u,v,ch,f)).  Exit code = failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "segconv_b200.h"

static int failures = 0;
#define CHECK(cond, what)                  \
  do {                                     \
    if (!(cond)) {                         \
      std::printf("FAIL %s\n", what);      \
      ++failures;                          \
    } else {                               \
      std::printf("PASS %s\n", what);      \
    }                                      \
  } while (0)

struct Spec {
  int n, cin, cout, k, p;
};

static std::vector<double> layer_ref(const std::vector<double>& x, int batch, const Spec& s, const std::vector<float>& k,
                                     const std::vector<float>& bias, int act) {
  const int out = 2 * s.n - 1 + 2 * s.p - s.k + 1;
  std::vector<double> y((size_t)batch * out * out * s.cout, 0.0);
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < s.n; ++i)
      for (int j = 0; j < s.n; ++j)
        for (int u = 0; u < s.k; ++u)
          for (int v = 0; v < s.k; ++v) {
            const int oy = 2 * i + s.p - u, ox = 2 * j + s.p - v;
            if (oy < 0 || oy >= out || ox < 0 || ox >= out) continue;
            for (int ch = 0; ch < s.cin; ++ch) {
              const double a = x[(((size_t)b * s.n + i) * s.n + j) * s.cin + ch];
              for (int f = 0; f < s.cout; ++f)
                y[(((size_t)b * out + oy) * out + ox) * s.cout + f] +=
                    a * k[(((size_t)u * s.k + v) * s.cin + ch) * s.cout + f];
            }
          }
  for (size_t e = 0; e < y.size(); ++e) {
    double v = y[e] + bias[e % s.cout];
    y[e] = act == 1 ? std::max(v, 0.0) : std::tanh(v);
  }
  return y;
}

int main() {
  const std::vector<Spec> specs = {{4, 64, 32, 3, 0}, {5, 32, 16, 4, 1}, {8, 16, 3, 3, 0}};
  const int batch = 7;
  std::mt19937_64 rng(2209);
  std::uniform_real_distribution<float> U(-1.0f, 1.0f);
  std::vector<std::vector<float>> ks, bs;
  std::vector<segconv_layer> layers;
  for (size_t l = 0; l < specs.size(); ++l) {
    const Spec& s = specs[l];
    std::vector<float> k((size_t)s.k * s.k * s.cin * s.cout), b((size_t)s.cout);
    for (float& v : k) v = 0.2f * U(rng);
    for (float& v : b) v = 0.1f * U(rng);
    ks.push_back(k);
    bs.push_back(b);
  }
  for (size_t l = 0; l < specs.size(); ++l) {
    const Spec& s = specs[l];
    segconv_layer L{};
    L.n_in = s.n, L.cin = s.cin, L.cout = s.cout, L.kh = L.kw = s.k, L.p_orig = s.p;
    L.h_kernel = ks[l].data();
    L.kernel_dtype = SEGCONV_F32;
    L.h_bias = bs[l].data();
    L.epilogue = SEGCONV_EPI_BIAS | (l + 1 < specs.size() ? SEGCONV_EPI_RELU : SEGCONV_EPI_TANH);
    L.math = SEGCONV_MATH_AUTO;
    layers.push_back(L);
  }
  std::vector<float> x((size_t)batch * 4 * 4 * 64);
  for (float& v : x) v = U(rng);
  std::vector<double> h(x.begin(), x.end());
  for (size_t l = 0; l < specs.size(); ++l)
    h = layer_ref(h, batch, specs[l], ks[l], bs[l], l + 1 < specs.size() ? 1 : 2);
  const int out = 2 * 8 - 3;
  std::vector<float> y((size_t)batch * out * out * 3, -7.0f);
  segconv_timing t{};
  segconv_status st = segconv_stack_run(layers.data(), (int)layers.size(), SEGCONV_F32, x.data(), batch, 0,
                                        y.data(), &t);
  if (st != SEGCONV_OK) std::printf("error: %s\n", segconv_last_error());
  CHECK(st == SEGCONV_OK, "segconv_stack_run on every visible GPU");
  double err = 0.0;
  for (size_t e = 0; e < y.size(); ++e)
    err = std::max(err, std::fabs(y[e] - h[e]) / std::max({std::fabs((double)y[e]), std::fabs(h[e]), 1.0}));
  std::printf("max scaled error %.3g over %zu outputs, %d GPU(s), compute %.3f ms, gather %.3f ms\n", err,
              y.size(), t.n_gpus, t.compute_ms, t.gather_ms);
  CHECK(err <= 1e-5, "stack output within the fp32 bar of the scatter reference");
  CHECK(t.n_gpus >= 1 && t.compute_ms > 0.0, "timing filled");
  // handle form: two forwards of different batch sizes
  segconv_stack* s = nullptr;
  st = segconv_stack_create(layers.data(), (int)layers.size(), SEGCONV_F32, batch, 0, &s);
  CHECK(st == SEGCONV_OK && s != nullptr, "segconv_stack_create");
  std::vector<float> y2(y.size(), 0.0f), y3(y.size(), 0.0f);
  CHECK(segconv_stack_forward(s, x.data(), batch, y2.data(), nullptr) == SEGCONV_OK, "forward (full batch)");
  CHECK(y2 == y, "handle forward == one-shot run");
  CHECK(segconv_stack_forward(s, x.data(), 3, y3.data(), nullptr) == SEGCONV_OK, "forward (3 images)");
  bool same = true;
  for (size_t e = 0; e < (size_t)3 * out * out * 3; ++e) same = same && y3[e] == y[e];
  CHECK(same, "a smaller batch gives the same images");
  CHECK(segconv_stack_forward(s, x.data(), batch + 1, y3.data(), nullptr) == SEGCONV_E_CONTRACT,
        "batch above max_batch is a contract error");
  segconv_stack_destroy(s);
  // chain mismatch: layer 1 expects 5x5x32
  layers[1].cin = 31;
  CHECK(segconv_stack_create(layers.data(), (int)layers.size(), SEGCONV_F32, batch, 0, &s) == SEGCONV_E_SHAPE,
        "a broken chain is a shape error");
  std::printf("%d failure(s)\n", failures);
  return failures;
}
