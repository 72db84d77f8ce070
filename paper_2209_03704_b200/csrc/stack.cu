// stack.cu -- batch-sharded multi-GPU driver for a chain of segregated
// transpose-convolution layers (include/segconv_b200.h, segconv_stack_*).
//
// The reference has one image per call and parallelises only over cout slices
// inside an image (proj/include/segconv/fused_tconv.hpp:101-147); the
// BASELINE's C5 workload is a four-layer generator over a batch of 1024.
// Images are independent, so the batch shards across GPUs with the weights
// replicated and no exchange between layers:
//   * creation: weights H2D on GPU 0, one ncclBroadcast per layer to the other
//     GPUs, segconv_segregate on every replica;
//   * forward: shard H2D per GPU (own stream), the layer chain, one
//     ncclAllGather of the output shards (padded to the largest shard so a
//     single collective moves them), GPU 0's full output D2H.
// One host thread drives every GPU (async launches on per-device streams);
// NCCL is loaded with dlopen so the library itself needs no libnccl at link
// time (a single-GPU stack never touches it).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "segconv_b200.h"

namespace segconv_b200 {
segconv_status set_error(segconv_status st, const char* msg);

namespace {

struct Nccl {
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.init_all = (decltype(n.init_all))dlsym(h, "ncclCommInitAll");
    n.destroy = (decltype(n.destroy))dlsym(h, "ncclCommDestroy");
    n.bcast = (decltype(n.bcast))dlsym(h, "ncclBroadcast");
    n.allgather = (decltype(n.allgather))dlsym(h, "ncclAllGather");
    n.group_start = (decltype(n.group_start))dlsym(h, "ncclGroupStart");
    n.group_end = (decltype(n.group_end))dlsym(h, "ncclGroupEnd");
    n.err = (decltype(n.err))dlsym(h, "ncclGetErrorString");
    n.ok = n.init_all && n.destroy && n.bcast && n.allgather && n.group_start && n.group_end && n.err;
  });
  return n;
}

size_t esize(int d) { return d == SEGCONV_F64 ? 8 : d == SEGCONV_BF16 ? 2 : 4; }
ncclDataType_t nccl_type(int d) {
  return d == SEGCONV_F64 ? ncclFloat64 : d == SEGCONV_BF16 ? ncclBfloat16 : ncclFloat32;
}

void shard(int batch, int g, int G, int* lo, int* hi) {
  const int base = batch / G, rem = batch % G;
  *lo = g * base + std::min(g, rem);
  *hi = *lo + base + (g < rem ? 1 : 0);
}

// A shard is uploaded in up to kMaxChunks slices of >= kChunkImages images
// on its own copy stream; the layer chain of slice c starts as soon as slice
// c has landed, so the host->device copy (the e2e bound: 33.5 MB for C5 at
// PCIe speed) overlaps the compute of the slices before it.
constexpr int kMaxChunks = 8, kChunkImages = 128;
int chunks_for(int b) { return std::max(1, std::min(kMaxChunks, b / kChunkImages)); }

struct Layer {
  segconv_layer desc;
  segconv_geometry geom;
  segconv_subkernels sks;
};

struct Replica {
  int dev = 0;
  cudaStream_t stream = nullptr;  // compute (and collectives)
  cudaStream_t copy = nullptr;    // shard upload, chunk by chunk
  cudaStream_t down = nullptr;    // one GPU: each chunk's output download, as soon as its chain ends
  cudaEvent_t ev[6] = {};      // h2d start, compute start, compute end, gather end, d2h end, h2d end
  cudaEvent_t chunk[kMaxChunks] = {};  // chunk c of the shard has landed
  cudaEvent_t done[kMaxChunks] = {};   // chunk c's chain has finished (one GPU: its download may start)
  void* x = nullptr;           // shard input
  std::vector<void*> acts;     // per-layer outputs (shard)
  std::vector<void*> kern;     // raw kernels (kept for the broadcast source / re-segregation)
  std::vector<void*> panels;   // segregated panels
  std::vector<float*> bias;
  void* gathered = nullptr;    // full-batch output (all-gathered)
  void* send = nullptr;        // padded shard of the last layer (all-gather source)
  ncclComm_t comm = nullptr;
};

}  // namespace
}  // namespace segconv_b200

using namespace segconv_b200;

struct segconv_stack {
  std::vector<Layer> layers;
  std::vector<Replica> reps;
  int dtype = SEGCONV_BF16;
  int max_batch = 0, max_shard = 0;
  size_t in_img = 0, out_img = 0;  // elements per image: input of layer 0, output of the last
};

static segconv_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return set_error(SEGCONV_E_CUDA, buf);
}
static segconv_status nccl_fail(ncclResult_t r, const char* what) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, nccl().err ? nccl().err(r) : "NCCL error");
  return set_error(SEGCONV_E_NCCL, buf);
}
#define CK(call, what)                                       \
  do {                                                       \
    const cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);       \
  } while (0)
#define NK(call, what)                                       \
  do {                                                       \
    const ncclResult_t r_ = (call);                          \
    if (r_ != ncclSuccess) return nccl_fail(r_, what);       \
  } while (0)

extern "C" {

void segconv_stack_destroy(segconv_stack* st) {
  if (!st) return;
  for (Replica& r : st->reps) {
    if (cudaSetDevice(r.dev) != cudaSuccess) continue;
    if (r.stream) cudaStreamSynchronize(r.stream);
    if (r.comm && nccl().ok) nccl().destroy(r.comm);
    cudaFree(r.x);
    for (void* p : r.acts) cudaFree(p);
    for (void* p : r.kern) cudaFree(p);
    for (void* p : r.panels) cudaFree(p);
    for (float* p : r.bias) cudaFree(p);
    cudaFree(r.gathered);
    cudaFree(r.send);
    for (cudaEvent_t e : r.ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : r.chunk)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : r.done)
      if (e) cudaEventDestroy(e);
    if (r.stream) cudaStreamDestroy(r.stream);
    if (r.copy) cudaStreamDestroy(r.copy);
    if (r.down) cudaStreamDestroy(r.down);
  }
  delete st;
}

static segconv_status stack_build(segconv_stack* st, const segconv_layer* layers, int n_layers, int dtype,
                                  int max_batch, int n_gpus) {
  if (!layers || n_layers < 1) return set_error(SEGCONV_E_CONTRACT, "a stack needs at least one layer");
  if (dtype != SEGCONV_F32 && dtype != SEGCONV_BF16)
    return set_error(SEGCONV_E_CONTRACT, "stack activations are f32 or bf16");
  if (max_batch < 1) return set_error(SEGCONV_E_CONTRACT, "max_batch must be >= 1");
  if (n_gpus < 0) return set_error(SEGCONV_E_CONTRACT, "n_gpus must be >= 0 (0: every visible GPU)");
  // chain checks first (host only): the geometry of each layer feeds the next
  for (int l = 0; l < n_layers; ++l) {
    Layer L{};
    L.desc = layers[l];
    const segconv_layer& d = layers[l];
    segconv_status s = segconv_tconv_geometry(d.n_in, d.kh, d.kw, d.p_orig, &L.geom);
    if (s != SEGCONV_OK) return s;
    if (d.cin < 1 || d.cout < 1) return set_error(SEGCONV_E_SHAPE, "layer channel counts must be >= 1");
    if (!d.h_kernel) return set_error(SEGCONV_E_CONTRACT, "layer kernel pointer is null");
    if ((d.epilogue & SEGCONV_EPI_BIAS) && !d.h_bias)
      return set_error(SEGCONV_E_CONTRACT, "bias epilogue requested without a bias pointer");
    if (l > 0) {
      const Layer& P = st->layers.back();
      if (P.geom.out_h != d.n_in || P.geom.out_w != d.n_in || P.desc.cout != d.cin) {
        char buf[160];
        snprintf(buf, sizeof buf, "layer %d output %dx%dx%d does not feed layer %d input %dx%dx%d", l - 1,
                 P.geom.out_h, P.geom.out_w, P.desc.cout, l, d.n_in, d.n_in, d.cin);
        return set_error(SEGCONV_E_SHAPE, buf);
      }
    }
    s = segconv_subkernels_for_math(d.kh, d.kw, d.cin, d.cout, d.p_orig, (segconv_dtype)dtype, d.math, &L.sks);
    if (s != SEGCONV_OK) return s;
    st->layers.push_back(L);
  }
  int devices = 0;
  CK(cudaGetDeviceCount(&devices), "stack: device count");
  if (n_gpus == 0) n_gpus = devices;
  if (n_gpus < 1 || n_gpus > devices) {
    char buf[128];
    snprintf(buf, sizeof buf, "stack: %d GPUs requested, %d visible", n_gpus, devices);
    return set_error(SEGCONV_E_CONTRACT, buf);
  }
  st->dtype = dtype;
  st->max_batch = max_batch;
  st->max_shard = (max_batch + n_gpus - 1) / n_gpus;
  const Layer& first = st->layers.front();
  const Layer& last = st->layers.back();
  st->in_img = (size_t)first.desc.n_in * first.desc.n_in * first.desc.cin;
  st->out_img = (size_t)last.geom.out_h * last.geom.out_w * last.desc.cout;
  const size_t es = esize(dtype);

  st->reps.resize((size_t)n_gpus);
  for (int g = 0; g < n_gpus; ++g) {
    Replica& r = st->reps[(size_t)g];
    r.dev = g;
    CK(cudaSetDevice(g), "stack: set device");
    CK(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking), "stack: stream");
    CK(cudaStreamCreateWithFlags(&r.copy, cudaStreamNonBlocking), "stack: copy stream");
    CK(cudaStreamCreateWithFlags(&r.down, cudaStreamNonBlocking), "stack: download stream");
    for (cudaEvent_t& e : r.ev) CK(cudaEventCreate(&e), "stack: event");
    for (cudaEvent_t& e : r.chunk) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "stack: event");
    for (cudaEvent_t& e : r.done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "stack: event");
    CK(cudaMalloc(&r.x, std::max<size_t>(1, st->max_shard * st->in_img * es)), "stack: input buffer");
    for (const Layer& L : st->layers) {
      void* a = nullptr;
      CK(cudaMalloc(&a, std::max<size_t>(1, (size_t)st->max_shard * L.geom.out_h * L.geom.out_w * L.desc.cout * es)),
         "stack: activation buffer");
      r.acts.push_back(a);
      void* k = nullptr;
      const size_t kb = (size_t)L.desc.kh * L.desc.kw * L.desc.cin * L.desc.cout * esize(L.desc.kernel_dtype);
      CK(cudaMalloc(&k, kb), "stack: kernel buffer");
      r.kern.push_back(k);
      void* pn = nullptr;
      CK(cudaMalloc(&pn, std::max<int64_t>(1, L.sks.total_elems) * esize(L.sks.dtype == SEGCONV_F16_SPLIT
                                                                              ? SEGCONV_BF16
                                                                              : L.sks.dtype)),
         "stack: panel buffer");
      r.panels.push_back(pn);
      float* b = nullptr;
      if (L.desc.epilogue & SEGCONV_EPI_BIAS) {
        CK(cudaMalloc(&b, L.desc.cout * sizeof(float)), "stack: bias buffer");
        CK(cudaMemcpyAsync(b, L.desc.h_bias, L.desc.cout * sizeof(float), cudaMemcpyHostToDevice, r.stream),
           "stack: bias upload");
      }
      r.bias.push_back(b);
    }
    CK(cudaMalloc(&r.send, std::max<size_t>(1, st->max_shard * st->out_img * es)), "stack: gather source");
    CK(cudaMalloc(&r.gathered, std::max<size_t>(1, (size_t)n_gpus * st->max_shard * st->out_img * es)),
       "stack: gathered output");
  }
  // weights: host -> GPU 0, then one broadcast per layer (replicated weights)
  CK(cudaSetDevice(0), "stack: set device");
  for (size_t l = 0; l < st->layers.size(); ++l) {
    const Layer& L = st->layers[l];
    const size_t kb = (size_t)L.desc.kh * L.desc.kw * L.desc.cin * L.desc.cout * esize(L.desc.kernel_dtype);
    CK(cudaMemcpyAsync(st->reps[0].kern[l], L.desc.h_kernel, kb, cudaMemcpyHostToDevice, st->reps[0].stream),
       "stack: kernel upload");
  }
  if (n_gpus > 1) {
    const Nccl& N = nccl();
    if (!N.ok) return set_error(SEGCONV_E_NCCL, "stack: libnccl.so.2 could not be loaded");
    std::vector<ncclComm_t> comms((size_t)n_gpus);
    std::vector<int> devs((size_t)n_gpus);
    for (int g = 0; g < n_gpus; ++g) devs[(size_t)g] = g;
    NK(N.init_all(comms.data(), n_gpus, devs.data()), "stack: ncclCommInitAll");
    for (int g = 0; g < n_gpus; ++g) st->reps[(size_t)g].comm = comms[(size_t)g];
    for (size_t l = 0; l < st->layers.size(); ++l) {
      const Layer& L = st->layers[l];
      const size_t n = (size_t)L.desc.kh * L.desc.kw * L.desc.cin * L.desc.cout;
      NK(N.group_start(), "stack: group");
      for (Replica& r : st->reps) {
        CK(cudaSetDevice(r.dev), "stack: set device");
        NK(N.bcast(st->reps[0].kern[l], r.kern[l], n, nccl_type(L.desc.kernel_dtype), 0, r.comm, r.stream),
           "stack: ncclBroadcast (weights)");
      }
      NK(N.group_end(), "stack: group");
    }
  }
  for (Replica& r : st->reps) {
    CK(cudaSetDevice(r.dev), "stack: set device");
    for (size_t l = 0; l < st->layers.size(); ++l) {
      const segconv_status s = segconv_segregate(r.kern[l], st->layers[l].desc.kernel_dtype, &st->layers[l].sks,
                                                 r.panels[l], r.stream);
      if (s != SEGCONV_OK) return s;
    }
  }
  for (Replica& r : st->reps) {
    CK(cudaSetDevice(r.dev), "stack: set device");
    CK(cudaStreamSynchronize(r.stream), "stack: setup");
  }
  return SEGCONV_OK;
}

segconv_status segconv_stack_create(const segconv_layer* layers, int n_layers, segconv_dtype dtype, int max_batch,
                                    int n_gpus, segconv_stack** out) {
  if (!out) return set_error(SEGCONV_E_CONTRACT, "stack output pointer is null");
  *out = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  segconv_stack* st = new segconv_stack();
  const segconv_status s = stack_build(st, layers, n_layers, dtype, max_batch, n_gpus);
  cudaSetDevice(prev);
  if (s != SEGCONV_OK) {
    segconv_stack_destroy(st);
    return s;
  }
  *out = st;
  return SEGCONV_OK;
}

int segconv_stack_gpus(const segconv_stack* st) { return st ? (int)st->reps.size() : 0; }

const void* segconv_stack_output(const segconv_stack* st, int gpu) {
  if (!st || gpu < 0 || gpu >= (int)st->reps.size()) return nullptr;
  return st->reps.size() > 1 ? st->reps[(size_t)gpu].gathered : st->reps[0].acts.back();
}

static segconv_status stack_forward(segconv_stack* st, const void* h_x, int batch, void* h_y, segconv_timing* tm) {
  const auto t0 = std::chrono::steady_clock::now();
  if (batch < 0 || batch > st->max_batch) {
    char buf[128];
    snprintf(buf, sizeof buf, "stack: batch %d outside [0, %d]", batch, st->max_batch);
    return set_error(SEGCONV_E_CONTRACT, buf);
  }
  if (batch == 0) return SEGCONV_OK;
  if (!h_x || !h_y) return set_error(SEGCONV_E_CONTRACT, "stack: null host buffer");
  const int G = (int)st->reps.size();
  const size_t es = esize(st->dtype);
  const int pad = (batch + G - 1) / G;  // all-gather unit: the largest shard
  for (int g = 0; g < G; ++g) {
    Replica& r = st->reps[(size_t)g];
    int lo, hi;
    shard(batch, g, G, &lo, &hi);
    const int b = hi - lo;
    CK(cudaSetDevice(r.dev), "stack: set device");
    CK(cudaEventRecord(r.ev[0], r.copy), "stack: event");
    const int C = chunks_for(b);
    for (int c = 0; c < C; ++c) {
      const int c0 = c * b / C, c1 = (c + 1) * b / C, nb = c1 - c0;
      if (nb <= 0) continue;
      CK(cudaMemcpyAsync((char*)r.x + (size_t)c0 * st->in_img * es,
                         (const char*)h_x + (size_t)(lo + c0) * st->in_img * es, (size_t)nb * st->in_img * es,
                         cudaMemcpyHostToDevice, r.copy),
         "stack: shard upload");
      CK(cudaEventRecord(r.chunk[c], r.copy), "stack: event");
      CK(cudaStreamWaitEvent(r.stream, r.chunk[c], 0), "stack: chunk wait");
      if (c == 0) CK(cudaEventRecord(r.ev[1], r.stream), "stack: event");
      const void* src = (const char*)r.x + (size_t)c0 * st->in_img * es;
      for (size_t l = 0; l < st->layers.size(); ++l) {
        const Layer& L = st->layers[l];
        void* dst = (char*)r.acts[l] + (size_t)c0 * L.geom.out_h * L.geom.out_w * L.desc.cout * es;
        const segconv_status s = segconv_transpose_conv_fused(
            src, (segconv_dtype)st->dtype, nb, L.desc.n_in, L.desc.cin, &L.sks, r.panels[l], &L.geom, r.bias[l],
            L.desc.epilogue, SEGCONV_MATH_AUTO, dst, (segconv_dtype)st->dtype, r.stream);
        if (s != SEGCONV_OK) return s;
        src = dst;
      }
      if (G == 1) {
        // one GPU: download this chunk's output while the next chunks upload and
        // compute (a third stream: the upload stream must not wait on compute)
        CK(cudaEventRecord(r.done[c], r.stream), "stack: event");
        CK(cudaStreamWaitEvent(r.down, r.done[c], 0), "stack: chunk done wait");
        CK(cudaMemcpyAsync((char*)h_y + (size_t)(lo + c0) * st->out_img * es, src, (size_t)nb * st->out_img * es,
                           cudaMemcpyDeviceToHost, r.down),
           "stack: chunk output download");
      }
    }
    if (b <= 0) CK(cudaEventRecord(r.ev[1], r.stream), "stack: event");
    CK(cudaEventRecord(r.ev[5], r.copy), "stack: event");
    CK(cudaEventRecord(r.ev[2], r.stream), "stack: event");
  }
  if (G > 1) {
    const Nccl& N = nccl();
    for (int g = 0; g < G; ++g) {  // padded shards: one all-gather moves them all
      Replica& r = st->reps[(size_t)g];
      int lo, hi;
      shard(batch, g, G, &lo, &hi);
      CK(cudaSetDevice(r.dev), "stack: set device");
      if (hi > lo)
        CK(cudaMemcpyAsync(r.send, r.acts.back(), (size_t)(hi - lo) * st->out_img * es, cudaMemcpyDeviceToDevice,
                           r.stream),
           "stack: gather staging");
    }
    NK(N.group_start(), "stack: group");
    for (Replica& r : st->reps) {
      CK(cudaSetDevice(r.dev), "stack: set device");
      NK(N.allgather(r.send, r.gathered, (size_t)pad * st->out_img, nccl_type(st->dtype), r.comm, r.stream),
         "stack: ncclAllGather (outputs)");
    }
    NK(N.group_end(), "stack: group");
  }  // one GPU: its last activation buffer is the full output
  for (Replica& r : st->reps) {
    CK(cudaSetDevice(r.dev), "stack: set device");
    CK(cudaEventRecord(r.ev[3], r.stream), "stack: event");
  }
  // GPU 0 holds every shard, each at g * pad images: compact them into h_y
  // (one GPU: the chunks are already on their way, on the download stream)
  Replica& r0 = st->reps[0];
  CK(cudaSetDevice(r0.dev), "stack: set device");
  if (G > 1) {
    for (int g = 0; g < G; ++g) {
      int lo, hi;
      shard(batch, g, G, &lo, &hi);
      if (hi > lo)
        CK(cudaMemcpyAsync((char*)h_y + (size_t)lo * st->out_img * es,
                           (const char*)r0.gathered + (size_t)g * pad * st->out_img * es,
                           (size_t)(hi - lo) * st->out_img * es, cudaMemcpyDeviceToHost, r0.stream),
           "stack: output download");
    }
    CK(cudaEventRecord(r0.ev[4], r0.stream), "stack: event");
  } else {
    CK(cudaEventRecord(r0.ev[4], r0.down), "stack: event");
  }
  double h2d = 0, comp = 0, gat = 0, d2h = 0;
  for (Replica& r : st->reps) {
    CK(cudaSetDevice(r.dev), "stack: set device");
    CK(cudaStreamSynchronize(r.stream), "stack: forward");
    CK(cudaStreamSynchronize(r.copy), "stack: forward");
    CK(cudaStreamSynchronize(r.down), "stack: forward");
    float a = 0, b = 0, c = 0;
    CK(cudaEventElapsedTime(&a, r.ev[0], r.ev[5]), "stack: timing");
    CK(cudaEventElapsedTime(&b, r.ev[1], r.ev[2]), "stack: timing");
    CK(cudaEventElapsedTime(&c, r.ev[2], r.ev[3]), "stack: timing");
    h2d = std::max(h2d, (double)a);
    comp = std::max(comp, (double)b);
    gat = std::max(gat, (double)c);
  }
  {
    float d = 0;
    CK(cudaSetDevice(r0.dev), "stack: set device");
    CK(cudaEventElapsedTime(&d, r0.ev[3], r0.ev[4]), "stack: timing");
    d2h = std::max(0.0, (double)d);  // one GPU: the downloads overlap compute, this is the tail after it
  }
  if (tm) {
    tm->n_gpus = G;
    tm->h2d_ms = h2d;
    tm->compute_ms = comp;
    tm->gather_ms = gat;
    tm->d2h_ms = d2h;
    tm->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return SEGCONV_OK;
}

segconv_status segconv_stack_forward(segconv_stack* st, const void* h_x, int batch, void* h_y,
                                     segconv_timing* timing) {
  if (!st) return set_error(SEGCONV_E_CONTRACT, "null stack handle");
  int prev = 0;
  cudaGetDevice(&prev);
  const segconv_status s = stack_forward(st, h_x, batch, h_y, timing);
  cudaSetDevice(prev);
  return s;
}

segconv_status segconv_stack_run(const segconv_layer* layers, int n_layers, segconv_dtype dtype, const void* h_x,
                                 int batch, int n_gpus, void* h_y, segconv_timing* timing) {
  segconv_stack* st = nullptr;
  segconv_status s = segconv_stack_create(layers, n_layers, dtype, std::max(1, batch), n_gpus, &st);
  if (s != SEGCONV_OK) return s;
  s = segconv_stack_forward(st, h_x, batch, h_y, timing);
  segconv_stack_destroy(st);
  return s;
}

}  // extern "C"
