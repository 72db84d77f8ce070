// segconv_b200 -- command-line caller of the GPU operators:
// the reference CLI's verify / bench / apply subcommands
// (proj/tools/segconv.cpp:53-66, 82-111, 195-228) over the drop-in host API
// (include/segconv_b200.hpp), with plain argv parsing instead of CLI11.
//
//   segconv_b200 verify [--cases N] [--seed S] [--n-min/--n-max/--k-min/--k-max/
//                        --p-min/--p-max/--c-min/--c-max V] [--inject-fault I]
//                        [--math exact|ffma|auto|bf16|f16x3]
//   segconv_b200 bench  [--preset flowers|gan:<model>|custom] [--size N --kernel n
//                        --padding P --cin C --cout F] [--reps R] [--seed S]
//                        [--format csv|json] [--out FILE]
//   segconv_b200 apply  --input X.sgc [--kernel ones|gaussian|random:<seed>|K.sgc]
//                        [--kernel-size n] [--padding P] [--variant naive|fused|
//                        fused_parallel] [--out Y.sgc]
//
// Images travel as SGC1 tensor files (the reference's PNM reader is out of
// scope).  verify draws its cases with the reference's generator and order
// (verify.hpp:66-122, mt19937_64 + uniform_int_distribution), so a seed names
// the same cases; the conventional path (transpose_conv_naive, EXACT math:
// the reference's own order) is the oracle, the segregated path runs in the
// selected math.  Exit codes follow the reference: 0 ok, 1 verify failure,
// 2 usage / contract / shape error, 3 I/O or parse error.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "segconv_b200.hpp"

namespace {

constexpr int kExitOk = 0, kExitVerifyFail = 1, kExitUsage = 2, kExitIo = 3;

struct Args {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string str(const std::string& k, const std::string& d) const { return has(k) ? kv.at(k) : d; }
  long long num(const std::string& k, long long d) const {
    if (!has(k)) return d;
    char* end = nullptr;
    const long long v = std::strtoll(kv.at(k).c_str(), &end, 10);
    if (!end || *end) throw segconv::ContractError("--" + k + " expects an integer, got '" + kv.at(k) + "'");
    return v;
  }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& known) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) throw segconv::ContractError("unexpected argument '" + s + "'");
    s = s.substr(2);
    if (std::find(known.begin(), known.end(), s) == known.end())
      throw segconv::ContractError("unknown option --" + s);
    if (i + 1 >= argc) throw segconv::ContractError("option --" + s + " needs a value");
    a.kv[s] = argv[++i];
  }
  return a;
}

segconv_math math_of(const std::string& m) {
  static const std::map<std::string, segconv_math> t = {{"auto", SEGCONV_MATH_AUTO}, {"ffma", SEGCONV_MATH_FFMA},
                                                        {"exact", SEGCONV_MATH_EXACT}, {"bf16", SEGCONV_MATH_BF16},
                                                        {"f16x3", SEGCONV_MATH_F16X3}};
  auto it = t.find(m);
  if (it == t.end()) throw segconv::ContractError("unknown math '" + m + "' (exact, ffma, auto, bf16, f16x3)");
  return it->second;
}

void emit(const std::string& text, const std::string& out_path) {
  if (out_path.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream out(out_path, std::ios::trunc);
  if (!out) throw segconv::IoError("cannot open " + out_path + " for writing");
  out << text;
  if (!out) throw segconv::IoError("write failure on " + out_path);
}

// ------------------------------------------------------------------ verify
std::string first_mismatch(const segconv::Tensor<float>& got, const segconv::Tensor<float>& want) {
  if (!got.same_shape(want)) return "shape mismatch";
  for (int y = 0; y < want.height(); ++y)
    for (int x = 0; x < want.width(); ++x)
      for (int ch = 0; ch < want.channels(); ++ch)
        if (got(y, x, ch) != want(y, x, ch))
          return "first mismatch at (" + std::to_string(y) + "," + std::to_string(x) + "," + std::to_string(ch) +
                 "): fused " + std::to_string(got(y, x, ch)) + ", reference " + std::to_string(want(y, x, ch));
  return "no elementwise mismatch";
}

int cmd_verify(const Args& a) {
  const int cases = (int)a.num("cases", 200);
  const std::uint64_t seed = (std::uint64_t)a.num("seed", 20240911);
  const int n_min = (int)a.num("n-min", 1), n_max = (int)a.num("n-max", 16);
  const int k_min = (int)a.num("k-min", 1), k_max = (int)a.num("k-max", 7);
  const int p_min = (int)a.num("p-min", 0), p_max = (int)a.num("p-max", 4);
  const int c_min = (int)a.num("c-min", 1), c_max = (int)a.num("c-max", 4);
  const int inject = (int)a.num("inject-fault", -1);
  const segconv_math math = math_of(a.str("math", "exact"));
  if (cases < 0) throw segconv::ContractError("case count must be >= 0");
  if (cases == 0) std::cout << "warning: --cases 0, nothing to verify\n";
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int> n_dist(n_min, n_max), p_dist(p_min, p_max), c_dist(c_min, c_max);
  std::uniform_int_distribution<int> value_dist(-8, 8);
  int failures = 0, run = 0;
  std::string first;
  for (int ci = 0; ci < cases; ++ci) {
    const int n = n_dist(rng), p = p_dist(rng);
    const int k_cap = std::min(k_max, 2 * n - 1 + 2 * p);
    std::uniform_int_distribution<int> k_dist(std::min(k_min, k_cap), k_cap);
    const int k = k_dist(rng), cin = c_dist(rng), cout = c_dist(rng);
    std::vector<float> xin((size_t)n * n * cin), kd((size_t)k * k * cin * cout);
    for (float& v : xin) v = (float)value_dist(rng);
    for (float& v : kd) v = (float)value_dist(rng);
    const auto input = segconv::Tensor<float>::from_data(n, n, cin, xin);
    const auto kernel = segconv::Kernel<float>::from_data(k, k, cin, cout, kd);
    // --inject-fault: sub-kernel element [0] of the first non-empty class gets
    // +1 (verify.hpp:95-101), i.e. source tap (u0, v0, 0, 0) of that class --
    // only the segregated operand sees it
    segconv::Kernel<float> kf = kernel;
    if (ci == inject)
      for (int q = 0; q < 4; ++q) {
        const int r = q >> 1, c = q & 1;
        if (segconv::active_tap_count(k, p, r) && segconv::active_tap_count(k, p, c)) {
          kf(segconv::first_active_tap(p, r), segconv::first_active_tap(p, c), 0, 0) += 1.0f;
          break;
        }
      }
    const auto geom = segconv::tconv_geometry(n, k, k, p);
    // fp32 data: "bf16" / "f16x3" both mean the split-fp16 tensor-core math,
    // which needs cin % 8 == 0 and taps in every parity class; other cases
    // (the generator's 1-4 channels, 1x1 kernels) run the EXACT SIMT path
    segconv_math m = math == SEGCONV_MATH_BF16 ? SEGCONV_MATH_F16X3 : math;
    const bool every_class = k <= 7 && segconv::active_tap_count(k, p, 0) && segconv::active_tap_count(k, p, 1);
    if (m == SEGCONV_MATH_F16X3 && (!every_class || cin % 8 != 0)) m = SEGCONV_MATH_EXACT;
    const auto sks = segconv::segregate(kf, p, m);
    const auto ref = segconv::transpose_conv_naive(input, kernel, p);
    const auto fused = segconv::transpose_conv_fused(input, sks, geom);
    ++run;
    if (!segconv::tensors_equal_exact(fused, ref)) {
      if (failures++ == 0)
        first = "first counterexample: case " + std::to_string(ci) + ", input " + std::to_string(n) + "x" +
                std::to_string(n) + "x" + std::to_string(cin) + ", kernel " + std::to_string(k) + "x" +
                std::to_string(k) + "x" + std::to_string(cin) + "x" + std::to_string(cout) + ", padding " +
                std::to_string(p) + ", seed " + std::to_string(seed) + "\n  " + first_mismatch(fused, ref) + "\n";
    }
  }
  std::cout << "verify: " << run << " cases, " << failures << " failures\n";
  if (failures) {
    std::cout << first;
    return kExitVerifyFail;
  }
  return kExitOk;
}

// ------------------------------------------------------------------- bench
std::vector<std::pair<std::string, segconv::LayerShape>> shapes_of(const Args& a) {
  const std::string preset = a.str("preset", "flowers");
  std::vector<std::pair<std::string, segconv::LayerShape>> out;
  if (preset == "flowers") {  // bench.hpp:118-124: 224^2 RGB -> 1, n = 3/4/5 at p = n - 2
    for (int n : {3, 4, 5})
      out.push_back({"flowers-" + std::to_string(n) + "x" + std::to_string(n), {224, 3, 1, n, n, n - 2}});
  } else if (preset.rfind("gan:", 0) == 0) {  // analysis.hpp:96-121: 4x4 kernels, p = 2
    static const std::map<std::string, std::vector<std::array<int, 4>>> gan = {
        {"dcgan", {{2, 4, 1024, 512}, {3, 8, 512, 256}, {4, 16, 256, 128}, {5, 32, 128, 3}}},
        {"artgan", {{2, 4, 512, 256}, {3, 8, 256, 128}, {4, 16, 128, 128}, {6, 32, 128, 3}}},
        {"gpgan", {{2, 4, 512, 256}, {3, 8, 256, 128}, {4, 16, 128, 64}, {5, 32, 64, 3}}},
        {"ebgan", {{2, 4, 2048, 1024}, {3, 8, 1024, 512}, {4, 16, 512, 256}, {5, 32, 256, 128},
                   {6, 64, 128, 64}, {7, 128, 64, 64}}}};
    const std::string id = preset.substr(4);
    auto it = gan.find(id);
    if (it == gan.end())
      throw segconv::ContractError("unknown GAN model '" + id + "' (known: dcgan, artgan, gpgan, ebgan)");
    for (const auto& l : it->second)
      out.push_back({id + "-L" + std::to_string(l[0]), {l[1], l[2], l[3], 4, 4, 2}});
  } else if (preset == "custom") {
    const int size = (int)a.num("size", 0), kernel = (int)a.num("kernel", 0), padding = (int)a.num("padding", -1);
    if (size < 1 || kernel < 1 || padding < 0)
      throw segconv::ContractError("custom preset needs --size, --kernel and --padding (with --cin/--cout optional)");
    out.push_back({"custom", {size, (int)a.num("cin", 1), (int)a.num("cout", 1), kernel, kernel, padding}});
  } else {
    throw segconv::ContractError("unknown preset '" + preset + "' (expected flowers, gan:<model>, or custom)");
  }
  return out;
}

template <typename F>
double time_median(F&& fn, int reps) {
  fn();  // warmup (bench.hpp:47-59 protocol)
  std::vector<double> t;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    fn();
    t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(t.begin(), t.end());
  return t.size() % 2 ? t[t.size() / 2] : 0.5 * (t[t.size() / 2 - 1] + t[t.size() / 2]);
}

int cmd_bench(const Args& a) {
  const int reps = (int)a.num("reps", 5);
  if (reps < 3) throw segconv::ContractError("benchmark repetitions must be >= 3");
  const std::uint64_t seed = (std::uint64_t)a.num("seed", 42);
  const std::string format = a.str("format", "csv");
  if (format != "csv" && format != "json") throw segconv::ContractError("--format is csv or json");
  struct Rec {
    std::string label, in, ker, variant;
    int p;
    double t, speedup;
  };
  std::vector<Rec> recs;
  for (const auto& [label, s] : shapes_of(a)) {
    std::cerr << "bench: " << label << " (input " << s.n_in << "x" << s.n_in << "x" << s.cin << ", kernel " << s.kh
              << "x" << s.kw << ", p=" << s.p_orig << ")\n";
    const auto geom = segconv::geometry_of(s);
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    std::vector<float> xin((size_t)s.n_in * s.n_in * s.cin), kd((size_t)s.kh * s.kw * s.cin * s.cout);
    for (float& v : xin) v = dist(rng);
    for (float& v : kd) v = dist(rng);
    const auto input = segconv::Tensor<float>::from_data(s.n_in, s.n_in, s.cin, xin);
    const auto kernel = segconv::Kernel<float>::from_data(s.kh, s.kw, s.cin, s.cout, kd);
    const auto sks = segconv::segregate(kernel, s.p_orig);  // untimed, as bench.hpp:83
    const double tn = time_median([&] { segconv::transpose_conv_naive(input, kernel, s.p_orig); }, reps);
    const double tf = time_median([&] { segconv::transpose_conv_fused(input, sks, geom); }, reps);
    const double tp = time_median([&] { segconv::transpose_conv_fused_parallel(input, sks, geom, 1); }, reps);
    const std::string in = std::to_string(s.n_in) + "x" + std::to_string(s.n_in) + "x" + std::to_string(s.cin);
    const std::string ker = std::to_string(s.kh) + "x" + std::to_string(s.kw) + "x" + std::to_string(s.cin) + "x" +
                            std::to_string(s.cout);
    recs.push_back({label, in, ker, "naive", s.p_orig, tn, 1.0});
    recs.push_back({label, in, ker, "fused", s.p_orig, tf, tn / tf});
    recs.push_back({label, in, ker, "fused_parallel", s.p_orig, tp, tn / tp});
  }
  std::string out;
  char buf[96];
  if (format == "csv") {
    out = "label,input_shape,kernel_shape,padding,variant,workers,wall_seconds,repetitions,speedup_vs_naive\n";
    for (const Rec& r : recs) {
      std::snprintf(buf, sizeof buf, ",%d,%s,1,%.9f,%d,%.4f\n", r.p, r.variant.c_str(), r.t, reps, r.speedup);
      out += r.label + "," + r.in + "," + r.ker + buf;
    }
  } else {
    out = "[\n";
    for (size_t i = 0; i < recs.size(); ++i) {
      const Rec& r = recs[i];
      std::snprintf(buf, sizeof buf, "%.9f, \"repetitions\": %d, \"speedup_vs_naive\": %.4f}", r.t, reps, r.speedup);
      out += (i ? ",\n" : "") + std::string("  {\"label\": \"") + r.label + "\", \"input_shape\": \"" + r.in +
             "\", \"kernel_shape\": \"" + r.ker + "\", \"padding\": " + std::to_string(r.p) + ", \"variant\": \"" +
             r.variant + "\", \"workers\": 1, \"wall_seconds\": " + buf;
    }
    out += "\n]\n";
  }
  emit(out, a.str("out", ""));
  return kExitOk;
}

// ------------------------------------------------------------------- apply
segconv::Kernel<float> apply_kernel(const Args& a, int channels) {
  const std::string spec = a.str("kernel", "ones");
  const int n = (int)a.num("kernel-size", 5);
  if (spec == "ones" || spec == "gaussian" || spec.rfind("random:", 0) == 0) {
    // channel-preserving presets (tools/segconv.cpp:140-185)
    if (n < 1) throw segconv::ContractError("--kernel-size must be >= 1");
    segconv::Kernel<float> k(n, n, channels, channels);
    if (spec == "ones") {
      for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v)
          for (int ch = 0; ch < channels; ++ch) k(u, v, ch, ch) = 1.0f / (float)(n * n);
    } else if (spec == "gaussian") {
      const double sigma = std::max(0.5, n / 3.0), mid = (n - 1) / 2.0;
      std::vector<double> g((size_t)n * n);
      double sum = 0;
      for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) sum += g[u * n + v] = std::exp(-((u - mid) * (u - mid) + (v - mid) * (v - mid)) /
                                                                    (2 * sigma * sigma));
      for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v)
          for (int ch = 0; ch < channels; ++ch) k(u, v, ch, ch) = (float)(g[u * n + v] / sum);
    } else {
      std::uint64_t seed = 0;
      try {
        seed = std::stoull(spec.substr(7));
      } catch (const std::exception&) {
        throw segconv::ContractError("bad kernel preset '" + spec + "': expected random:<integer seed>");
      }
      std::mt19937_64 rng(seed);
      std::uniform_real_distribution<float> dist(-0.5f, 0.5f);
      for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v)
          for (int ch = 0; ch < channels; ++ch)
            for (int f = 0; f < channels; ++f) k(u, v, ch, f) = dist(rng);
    }
    return k;
  }
  // a tensor file kh x kw x cin: one output channel mixing all channels
  const auto t = segconv::load_tensor<float>(spec);
  if (t.channels() != channels)
    throw segconv::ContractError("kernel file has " + std::to_string(t.channels()) + " channels, image has " +
                                 std::to_string(channels));
  return segconv::Kernel<float>::from_data(t.height(), t.width(), t.channels(), 1,
                                           std::vector<float>(t.data(), t.data() + t.size()));
}

int cmd_apply(const Args& a) {
  if (!a.has("input")) throw segconv::ContractError("apply needs --input <tensor.sgc>");
  const auto image = segconv::load_tensor<float>(a.str("input", ""));
  if (image.height() != image.width())
    throw segconv::ContractError("transpose conv expects a square image, got " + std::to_string(image.height()) +
                                 "x" + std::to_string(image.width()));
  const auto kernel = apply_kernel(a, image.channels());
  const int p = (int)a.num("padding", 2);
  const std::string variant = a.str("variant", "fused");
  segconv::Tensor<float> result;
  if (variant == "naive") {
    result = segconv::transpose_conv_naive(image, kernel, p);
  } else if (variant == "fused") {
    result = segconv::transpose_conv_fused(image, kernel, p);
  } else if (variant == "fused_parallel") {
    const auto geom = segconv::tconv_geometry(image.height(), kernel.kh(), kernel.kw(), p);
    result = segconv::transpose_conv_fused_parallel(image, segconv::segregate(kernel, p), geom,
                                                    (int)a.num("workers", 1));
  } else {
    throw segconv::ContractError("unknown variant '" + variant + "' (naive, fused, fused_parallel)");
  }
  const std::string out = a.str("out", "out.sgc");
  segconv::save_tensor(result, out);
  std::cout << "apply: " << image.height() << "x" << image.width() << "x" << image.channels() << " -> "
            << result.height() << "x" << result.width() << "x" << result.channels() << ", tensor written to " << out
            << "\n";
  return kExitOk;
}

void usage() {
  std::cerr << "usage: segconv_b200 <verify|bench|apply> [--option value ...]\n"
               "  verify --cases --seed --n-min --n-max --k-min --k-max --p-min --p-max --c-min --c-max\n"
               "         --inject-fault --math\n"
               "  bench  --preset flowers|gan:<model>|custom --size --kernel --padding --cin --cout --reps\n"
               "         --seed --format csv|json --out\n"
               "  apply  --input X.sgc --kernel ones|gaussian|random:<seed>|K.sgc --kernel-size --padding\n"
               "         --variant naive|fused|fused_parallel --workers --out\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return kExitUsage;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "verify")
      return cmd_verify(parse(argc, argv, 2,
                              {"cases", "seed", "n-min", "n-max", "k-min", "k-max", "p-min", "p-max", "c-min", "c-max",
                               "inject-fault", "math"}));
    if (cmd == "bench")
      return cmd_bench(parse(argc, argv, 2,
                             {"preset", "size", "kernel", "padding", "cin", "cout", "workers", "reps", "seed", "format",
                              "out"}));
    if (cmd == "apply")
      return cmd_apply(parse(argc, argv, 2,
                             {"input", "kernel", "kernel-size", "padding", "variant", "workers", "out"}));
    usage();
    return kExitUsage;
  } catch (const segconv::ParseError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitIo;
  } catch (const segconv::IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitIo;
  } catch (const segconv::ShapeError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const segconv::ContractError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitVerifyFail;
  }
}
