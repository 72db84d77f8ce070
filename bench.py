#!/usr/bin/env python
"""Benchmark of the segregated transpose convolution on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl segconv|reference]

A step is one pass of the hot path (transpose_conv_fused, or the C5 stack)
over one batch of synthetic input resident in HBM.  Weights are segregated
once, untimed, as the reference bench does (proj/include/segconv/bench.hpp:83).
Each timed step is bracketed by CUDA events on the launching stream; L2 is
flushed (256 MiB write) between steps outside the events.  Multi-GPU: one
process per GPU (torchrun), max over ranks.  Prints ONE JSON line on rank 0.

Metric (BASELINE.json): useful GMAC/s (count_ops_fused numerator, reference
analysis.hpp:48-67) with HBM GB/s / tensor TFLOP/s as a fraction of the
measured roofline, vs the GPU upsample+conv path.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "useful GMAC/s & HBM GB/s (frac of roofline) vs upsample+conv, 1/2/4/8 B200"

# BASELINE.json configs.  dist: u = U[-1,1]; n = N(0,1); he = N(0, sqrt(2/(cin*k*k)));
# n02 = N(0, 0.02).
CONFIGS = {
    "C1": dict(batch=1, n=32, cin=1, cout=1, k=3, p=0, dtype="f32", xd="u", wd="u", act=None,
               desc="single-channel fp32, 1x32x32x1 -> 61x61x1, n=3"),
    "C2": dict(batch=16, n=64, cin=64, cout=32, k=3, p=0, dtype="f32", xd="u", wd="he", act=None,
               desc="multi-channel fp32, 16x64x64x64 -> 16x125x125x32, n=3"),
    "C3": dict(batch=128, n=16, cin=512, cout=256, k=4, p=0, dtype="bf16", xd="n", wd="n02",
               act=None, desc="DCGAN-style bf16, 128x16x16x512 -> 128x28x28x256, n=4"),
    # SURVEY 8(d) C3 "fp32-storage variant": the same layer in the reference's own dtype
    "C3f32": dict(batch=128, n=16, cin=512, cout=256, k=4, p=0, dtype="f32", xd="n", wd="n02",
                  act=None, desc="C3 layer in fp32 storage (split-fp16 tensor-core math), not a BASELINE line"),
    "C4": dict(batch=32, n=256, cin=64, cout=3, k=5, p=0, dtype="f32", xd="u", wd="n02",
               act="tanh", desc="low-channel fp32 + tanh, 32x256x256x64 -> 32x507x507x3, n=5"),
    "C5": dict(batch=1024, stack=True, dtype="bf16",
               desc="4-layer bf16 generator stack, batch 1024 sharded, 4->5->7->11->19"),
    # single layers of the C5 stack (diagnostics: --config C5a .. C5d)
    # GAN generator presets (reference analysis.hpp:96-114, bench.hpp:118-124 `gan:<model>`):
    # every layer 4x4 at p = 2 (out = 2N), bf16 chain, batch 64; not BASELINE configs
    "gan:dcgan": dict(batch=64, stack=True, gan="dcgan", dtype="bf16",
                      desc="DCGAN generator 4->64, 1024->3 channels, batch 64"),
    "gan:artgan": dict(batch=64, stack=True, gan="artgan", dtype="bf16",
                       desc="Art-GAN generator 4->64, 512->3 channels, batch 64"),
    "gan:gpgan": dict(batch=64, stack=True, gan="gpgan", dtype="bf16",
                      desc="GP-GAN generator 4->64, 512->3 channels, batch 64"),
    "gan:ebgan": dict(batch=64, stack=True, gan="ebgan", dtype="bf16",
                      desc="EB-GAN generator 4->256, 2048->64 channels, batch 64"),
    "C5a": dict(batch=1024, n=4, cin=1024, cout=512, k=3, p=0, dtype="bf16", xd="n", wd="n02",
                act="relu", desc="C5 layer a: 1024x4x4x1024 -> 5x5x512"),
    "C5b": dict(batch=1024, n=5, cin=512, cout=256, k=3, p=0, dtype="bf16", xd="n", wd="n02",
                act="relu", desc="C5 layer b: 1024x5x5x512 -> 7x7x256"),
    "C5c": dict(batch=1024, n=7, cin=256, cout=128, k=3, p=0, dtype="bf16", xd="n", wd="n02",
                act="relu", desc="C5 layer c: 1024x7x7x256 -> 11x11x128"),
    "C5d": dict(batch=1024, n=11, cin=128, cout=3, k=3, p=0, dtype="bf16", xd="n", wd="n02",
                act="tanh", desc="C5 layer d: 1024x11x11x128 -> 19x19x3"),
}
SEED = 20240911


_DIST = [False]


def dist_on():
    """The GPU arm runs over a process group (NCCL): at world size > 1, or at
    world size 1 under --dist (the driver's launch form exercised end to end on
    a one-GPU box: NCCL init, the weight broadcast, the max-over-ranks
    reduction and the all-gather, each a one-rank collective)."""
    return _DIST[0]


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def gen(shape, dist, rng, fan_in=1):
    if dist == "u":
        return rng.uniform(-1.0, 1.0, shape).astype(np.float32)
    if dist == "n":
        return rng.standard_normal(shape, dtype=np.float32)
    if dist == "he":
        return (rng.standard_normal(shape, dtype=np.float32) * np.float32(np.sqrt(2.0 / fan_in)))
    if dist == "n02":
        return rng.standard_normal(shape, dtype=np.float32) * np.float32(0.02)
    raise ValueError(dist)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"], "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "src": "fallback"}


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            self.p.wait(timeout=5)

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip() == "Active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


# --------------------------------------------------------------- problem
class Layer:
    """One segregated transpose conv (C1-C4) with host + device buffers."""

    def __init__(self, cfg, rank, torch, sc, dev, world):
        self.cfg = cfg
        rng = np.random.default_rng(SEED + 7919 * rank)
        b, n, cin, cout, k, p = (cfg[x] for x in ("batch", "n", "cin", "cout", "k", "p"))
        self.x_host = gen((b, n, n, cin), cfg["xd"], rng)
        krng = np.random.default_rng(SEED)
        self.k_host = gen((k, k, cin, cout), cfg["wd"], krng, fan_in=cin * k * k)
        self.tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
        kd = torch.from_numpy(self.k_host).to(dev)
        if dist_on():  # weights replicated from rank 0 (NCCL broadcast, untimed)
            torch.distributed.broadcast(kd, src=0)
        self.kd = kd.to(self.tdt)
        self.xd = torch.from_numpy(self.x_host).to(dev, self.tdt)
        self.g = sc.tconv_geometry(n, k, k, p)
        self.sks = sc.segregate(self.kd, p, math="auto")
        self.math = {v: k for k, v in sc.MATHS.items()}[self.sks.math]
        self.y = torch.empty((b, self.g.out_h, self.g.out_w, cout), dtype=self.tdt, device=dev)
        self.x_pinned = torch.from_numpy(self.x_host).to(self.tdt).pin_memory()
        self.y_pinned = torch.empty(self.y.shape, dtype=self.tdt).pin_memory()
        self.sc = sc
        self.macs = sc.count_ops_fused(sc.LayerShape(n, cin, cout, k, k, p)).mults * b
        e = self.xd.element_size()
        self.alg_bytes = (self.xd.numel() + self.kd.numel() + self.y.numel()) * e
        self.launches_per_step = 1
        # tensor-bound when the arithmetic intensity clears the ridge point; a
        # split-fp16 layer's tensor peak is a third of bf16 (3 MMAs per product)
        ai = 2.0 * self.macs / max(1, self.alg_bytes)
        pk = peaks()
        split = self.math == "f16x3"
        self.bound = "tensor" if self.math in ("bf16", "tf32") or \
            (split and ai > pk["bf16"] * 1e3 / 3 / pk["hbm"]) else "hbm"
        self.tensor_peak_div = 3.0 if split else 1.0

    def step(self):
        self.sc.transpose_conv_fused(self.xd, self.sks, self.g, activation=self.cfg["act"],
                                     out=self.y)

    def step_e2e(self):
        """Public API with host buffers (C ABI segconv_transpose_conv_fused_host): the
        step's input H2D, compute and result D2H, pipelined over batch slices."""
        self.sc.transpose_conv_fused(self.x_pinned, self.sks, self.g, activation=self.cfg["act"],
                                     out=self.y_pinned, staging=(self.xd, self.y), sync=False)

    def e2e_bytes(self):
        return self.x_pinned.numel() * self.x_pinned.element_size(), \
            self.y_pinned.numel() * self.y_pinned.element_size()

    def conventional(self, torch, steps, flush):
        """GPU upsample+conv (reference transpose_conv_naive) on the same data."""
        cfg = self.cfg
        ws_need = (cfg["batch"] * self.g.up_h ** 2 * cfg["cin"] * self.xd.element_size())
        if ws_need > 24 * 2 ** 30:
            return None
        xf = self.xd  # same dtype as the fused path (bf16 -> tensor-core conv2d_valid)
        kf = self.kd
        ws = torch.empty(ws_need, dtype=torch.uint8, device="cuda")
        ts = []
        for i in range(steps + 1):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            self.sc.transpose_conv_naive(xf, kf, cfg["p"], activation=cfg["act"], workspace=ws)
            b.record()
            b.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        return {"value": round(self.macs / (ms * 1e-3) / 1e9, 2), "ms_per_step": round(ms, 4),
                "what": "GPU upsample2x+pad then valid correlation (segconv_transpose_conv_naive; "
                        + self.sc.last_path() + " correlation)"}

    def cudnn(self, torch, steps, flush):
        """Library context: torch conv_transpose2d (cuDNN) on the same problem, NCHW."""
        cfg = self.cfg
        k = torch.from_numpy(self.k_host).cuda().to(self.tdt)
        W = k.permute(2, 3, 0, 1).flip(2, 3).contiguous()
        xn = self.xd.permute(0, 3, 1, 2).contiguous()
        ts = []
        for i in range(steps + 1):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            torch.nn.functional.conv_transpose2d(xn, W, stride=2, padding=cfg["k"] - 1 - cfg["p"])
            b.record()
            b.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        return {"value": round(self.macs / (ms * 1e-3) / 1e9, 2), "ms_per_step": round(ms, 4),
                "what": "torch.nn.functional.conv_transpose2d (cuDNN), NCHW input, not ours"}

    def cpu_sample(self, workers):
        """Reference CPU path on a bounded sample of the batch: (out, secs, images)."""
        import oracle
        nimg = min(self.cfg["batch"], max(1, 2 * workers))
        x = self.x_host[:nimg]
        k = self.k_host
        if self.cfg["dtype"] == "bf16":
            x, k = oracle.bf16_round(x), oracle.bf16_round(k)
        mode = 1  # images across threads, reference's sequential transpose_conv_fused each
        if oracle.ref_available():
            _, secs = oracle.ref_time_fused_batch(mode, x, k, self.cfg["p"], workers)
            return secs, nimg, "reference"
        t0 = time.perf_counter()
        oracle.tconv_fused(x, k, self.cfg["p"])
        return time.perf_counter() - t0, nimg, "port"


    def parity(self):
        """Two sampled images of the timed output against the oracle (the
        reference's segregated path restated in C, pinned to its goldens)."""
        import oracle
        b = self.cfg["batch"]
        idx = sorted({0, b - 1})
        x, k = self.x_host[idx], self.k_host
        if self.cfg["dtype"] == "bf16":
            x, k = oracle.bf16_round(x), oracle.bf16_round(k)
        want = oracle.tconv_fused(x, k, self.cfg["p"])
        if self.cfg["act"] == "tanh":
            want = np.tanh(want)
        elif self.cfg["act"] == "relu":
            want = np.maximum(want, 0)
        got = self.y[idx].float().cpu().numpy()
        tol = 1e-2 if self.cfg["dtype"] == "bf16" else 1e-5
        return {"max_scaled_err": scaled_err(got, want), "tol": tol, "images": idx,
                "oracle": "oracle.tconv_fused (C port, pinned)"}


class LayerBackward(Layer):
    """`--pass backward`: the layer's backward pass (reference netdemo/layers.hpp:171-211,
    input + kernel gradients) on the same synthetic layer, output gradient ~ N(0, 1).
    Useful MACs = 2 x the forward's (every forward product has one input-gradient
    and one kernel-gradient product)."""

    def __init__(self, cfg, rank, torch, sc, dev, world):
        super().__init__(cfg, rank, torch, sc, dev, world)
        rng = np.random.default_rng(SEED + 31 + rank)
        self.gy_host = rng.standard_normal(tuple(self.y.shape), dtype=np.float32)
        self.gyd = torch.from_numpy(self.gy_host).to(dev, self.tdt)
        self.gy_pinned = torch.from_numpy(self.gy_host).to(self.tdt).pin_memory()
        self.macs *= 2
        e = self.xd.element_size()
        self.alg_bytes = (2 * self.xd.numel() + self.kd.numel() + self.gyd.numel()) * e + \
            self.kd.numel() * 4
        self.torch = torch
        self.world = world
        self.launches_per_step = 2
        self.gx_pinned = torch.empty(self.xd.shape, dtype=self.tdt).pin_memory()
        self.gk_pinned = torch.empty(self.kd.shape, dtype=torch.float32).pin_memory()

    def step(self):
        if dist_on():
            # data-parallel step: the kernel gradient's all-reduce (NCCL) runs while
            # the input-gradient kernel computes (paper_2209_03704_b200/dp.py)
            _, gk = self.sc.transpose_conv_fused_backward(self.xd, self.kd, self.cfg["p"], self.gyd,
                                                          input_grad=False)
            work = self.torch.distributed.all_reduce(gk, async_op=True)
            gx, _ = self.sc.transpose_conv_fused_backward(self.xd, self.kd, self.cfg["p"], self.gyd,
                                                          kernel_grad=False)
            work.wait()
            self.math = "bwd:dp (" + self.sc.last_path() + ", kernel grad all-reduced)"
            self.gx_last = gx
            return
        gx, _ = self.sc.transpose_conv_fused_backward(self.xd, self.kd, self.cfg["p"], self.gyd)
        self.math = self.sc.last_path()  # e.g. "bwd:tc-pair+tc-pair"
        self.gx_last = gx

    def parity(self):
        """Input gradient of two sampled images against the oracle backward
        (reference net::FusedTConv::backward restated; per image it depends on
        that image's output gradient only)."""
        import oracle
        b = self.cfg["batch"]
        idx = sorted({0, b - 1})
        x, k, gy = self.x_host[idx], self.k_host, self.gy_host[idx]
        if self.cfg["dtype"] == "bf16":
            x, k, gy = oracle.bf16_round(x), oracle.bf16_round(k), oracle.bf16_round(gy)
        wx, _ = oracle.tconv_backward(x, k, self.cfg["p"], gy)
        got = self.gx_last[idx].float().cpu().numpy()
        tol = 1e-2 if self.cfg["dtype"] == "bf16" else 1e-5
        return {"max_scaled_err": scaled_err(got, wx), "tol": tol, "images": idx,
                "what": "input gradient", "oracle": "oracle.tconv_backward (C port, pinned)"}

    def f16x3_leg(self, torch, steps, flush):
        """fp32 layers: the step with math="f16x3" given explicitly (the input
        gradient on the tensor cores in split-fp16 math where the shape allows,
        the kernel gradient FFMA) -- AUTO takes the same path behind its
        device-side range guard -- timed with events around each call."""
        import oracle
        ts = []
        for i in range(steps + 2):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gx, _ = self.sc.transpose_conv_fused_backward(self.xd, self.kd, self.cfg["p"], self.gyd, math="f16x3")
            b.record()
            b.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        path = self.sc.last_path()
        idx = sorted({0, self.cfg["batch"] - 1})
        wx, _ = oracle.tconv_backward(self.x_host[idx], self.k_host, self.cfg["p"], self.gy_host[idx])
        err = scaled_err(gx[idx].float().cpu().numpy(), wx)
        ms = statistics.median(ts)
        return {"ms": round(ms, 5), "value": round(self.macs / (ms * 1e-3) / 1e9, 2), "unit": "useful GMAC/s",
                "path": path, "parity": {"max_scaled_err": err, "tol": 1e-5, "images": idx},
                "what": "math=\"f16x3\" explicitly (AUTO takes the same guarded path)"}

    e2e_what = ("segconv.transpose_conv_fused_backward from pinned host buffers: x and gy "
                "uploaded, both gradients read back, all on the launching stream")

    def step_e2e(self):
        """Public API from host buffers: x and gy uploaded, both gradients read back."""
        xd = self.x_pinned.to(self.xd.device, non_blocking=True)
        gyd = self.gy_pinned.to(self.xd.device, non_blocking=True)
        gx, gk = self.sc.transpose_conv_fused_backward(xd, self.kd, self.cfg["p"], gyd)
        self.gx_pinned.copy_(gx, non_blocking=True)
        self.gk_pinned.copy_(gk, non_blocking=True)

    def e2e_bytes(self):
        return (self.x_pinned.numel() + self.gy_pinned.numel()) * self.x_pinned.element_size(), \
            self.gx_pinned.numel() * self.gx_pinned.element_size() + self.gk_pinned.numel() * 4

    def conventional(self, torch, steps, flush):
        return None

    def cudnn(self, torch, steps, flush):
        """Library context: torch's conv_transpose2d backward (cuDNN dgrad + wgrad), NCHW."""
        cfg = self.cfg
        k = torch.from_numpy(self.k_host).cuda().to(self.tdt)
        W = k.permute(2, 3, 0, 1).flip(2, 3).contiguous().requires_grad_(True)
        xn = self.xd.permute(0, 3, 1, 2).contiguous().requires_grad_(True)
        y = torch.nn.functional.conv_transpose2d(xn, W, stride=2, padding=cfg["k"] - 1 - cfg["p"])
        g = self.gyd.permute(0, 3, 1, 2).contiguous()
        ts = []
        for i in range(steps + 1):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            torch.autograd.grad(y, (xn, W), g, retain_graph=True)
            b.record()
            b.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        return {"value": round(self.macs / (ms * 1e-3) / 1e9, 2), "ms_per_step": round(ms, 4),
                "what": "torch conv_transpose2d backward (cuDNN dgrad + wgrad), NCHW, not ours"}

    def cpu_sample(self, workers):
        import oracle
        nimg = min(self.cfg["batch"], max(1, workers))
        x, k, gy = self.x_host[:nimg], self.k_host, self.gy_host[:nimg]
        if self.cfg["dtype"] == "bf16":
            x, k, gy = oracle.bf16_round(x), oracle.bf16_round(k), oracle.bf16_round(gy)
        if oracle.ref_available():
            _, _, secs = oracle.ref_time_backward(x, k, self.cfg["p"], gy, workers)
            return secs, nimg, "reference"
        t0 = time.perf_counter()
        oracle.tconv_backward(x, k, self.cfg["p"], gy)
        return time.perf_counter() - t0, nimg, "port"


class Stack:
    """BASELINE C5: four-layer bf16 generator stack, batch 1024 sharded over ranks
    (ShardedStack: weights broadcast once from rank 0, all-gather of the outputs)."""

    def __init__(self, cfg, rank, world, torch, sc, dev, batch=None, with_capi=True):
        from paper_2209_03704_b200 import stack as st
        self.torch, self.sc, self.st = torch, sc, st
        self.cfg = cfg
        self.world = world
        self.specs = stack_specs(cfg)
        krng = np.random.default_rng(SEED)
        self.k_host = [gen((s.k, s.k, s.cin, s.cout), "n02", krng) for s in self.specs]
        ks = [torch.from_numpy(k).to(dev) for k in self.k_host]
        gb = cfg["batch"] if batch is None else batch
        self.global_batch = gb
        s0 = self.specs[0]
        rng = np.random.default_rng(SEED + 1)
        xall = rng.standard_normal((gb, s0.n_in, s0.n_in, s0.cin), dtype=np.float32)
        if dist_on():
            self.sharded = st.ShardedStack(self.specs, ks, gb, act_dtype=torch.bfloat16)
            self.stack = self.sharded.local
            self.lo, self.hi = self.sharded.lo, self.sharded.hi
        else:
            self.sharded = None
            self.stack = st.GeneratorStack(self.specs, ks, gb, act_dtype=torch.bfloat16)
            self.lo, self.hi = 0, gb
        self.x_host = xall[self.lo:self.hi]
        self.stack.x.copy_(torch.from_numpy(self.x_host))
        self.math = "+".join({v: k for k, v in sc.MATHS.items()}[s.math] for s in self.stack.sks)
        self.stack.capture()
        self.macs = self.stack.useful_macs()
        self.alg_bytes = self.stack.algorithmic_bytes()
        self.launches_per_step = len(self.specs)
        self.bound = "tensor"
        self.x_pinned = torch.from_numpy(self.x_host).to(torch.bfloat16).pin_memory()
        self.y_pinned = torch.empty(self.stack.out.shape, dtype=torch.bfloat16).pin_memory()
        self.paths = []
        # e2e at one process: the C ABI's stack driver (segconv_stack_forward,
        # host buffers in and out: shard H2D, the chain, output D2H)
        self.capi = st.MultiGPUStack(self.specs, [torch.from_numpy(k) for k in self.k_host], gb,
                                     n_gpus=1) if world == 1 and with_capi else None
        self.e2e_what = ("C ABI segconv_stack_forward (host buffers; H2D + 4 layers + D2H, synchronous)"
                         if self.capi is not None else
                         "per rank: pinned H2D of the shard, the stack graph, D2H of the shard output")

    def step(self):
        self.stack.forward()

    def step_e2e(self):
        if self.capi is not None:
            self.capi.forward(self.x_pinned, out=self.y_pinned)
            return
        self.stack.x.copy_(self.x_pinned, non_blocking=True)
        self.stack.forward()
        self.y_pinned.copy_(self.stack.out, non_blocking=True)

    def e2e_bytes(self):
        return self.x_pinned.numel() * 2, self.y_pinned.numel() * 2

    def gather(self):
        """The path's one exchange: all-gather of the output shards (NCCL)."""
        return self.sharded.gather() if self.sharded is not None else self.stack.out

    def layer_times(self, steps, flush):
        """Per-layer device time (eager launches, CUDA events between layers on the
        launching stream): the dominant kernel of the step and its roofline."""
        torch = self.torch
        st = self.stack
        per = [[] for _ in self.specs]
        for i in range(steps + 1):
            flush()
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(self.specs) + 1)]
            src = st.x
            evs[0].record()
            paths = []
            for li, (s, g, sks, dst) in enumerate(zip(st.specs, st.geoms, st.sks, st.acts)):
                self.sc.transpose_conv_fused(src, sks, g, activation=s.activation, out=dst)
                paths.append(self.sc.last_path())
                evs[li + 1].record()
                src = dst
            torch.cuda.synchronize()
            if i:
                for li in range(len(self.specs)):
                    per[li].append(evs[li].elapsed_time(evs[li + 1]))
            self.paths = paths
        out = []
        pk = peaks()
        for li, (s, g) in enumerate(zip(st.specs, st.geoms)):
            ms = statistics.mean(per[li])
            macs = self.sc.count_ops_fused(self.sc.LayerShape(s.n_in, s.cin, s.cout, s.k, s.k, s.p)).mults \
                * st.batch
            byts = (st.batch * (s.n_in ** 2 * s.cin + g.out_h * g.out_w * s.cout) + s.k * s.k * s.cin * s.cout) * 2
            ai = 2.0 * macs / byts
            tensor = ai > pk["bf16"] * 1e3 / pk["hbm"]
            ach = (2.0 * macs / (ms * 1e-3) / 1e12) if tensor else (byts / (ms * 1e-3) / 1e9)
            peak = pk["bf16"] if tensor else pk["hbm"]
            out.append({"layer": "abcdefgh"[li], "shape": f"{s.n_in}x{s.n_in}x{s.cin}->{g.out_h}x{g.out_w}x{s.cout}",
                        "path": paths[li] if li < len(self.paths) else None, "ms": round(ms, 4),
                        "useful_macs": macs, "alg_bytes": byts,
                        "bound": "tensor" if tensor else "hbm", "achieved": round(ach, 1),
                        "unit": "TFLOP/s" if tensor else "GB/s", "peak": peak,
                        "frac": round(ach / peak, 4)})
        return out

    def conventional(self, torch, steps, flush):
        return None

    def cudnn(self, torch, steps, flush):
        return None

    def cpu_sample(self, workers):
        import oracle
        nimg = min(self.hi - self.lo, max(1, 2 * workers))
        x = oracle.bf16_round(self.x_host[:nimg])
        t0 = time.perf_counter()
        secs = 0.0
        kind = "reference" if oracle.ref_available() else "port"
        for s, k in zip(self.specs, self.k_host):
            kb = oracle.bf16_round(k)
            if kind == "reference":
                y, dt = oracle.ref_time_fused_batch(1, x, kb, s.p, workers)
                secs += dt
            else:
                y = oracle.tconv_fused(x, kb, s.p)
            y = np.maximum(y, 0) if s.activation == "relu" else np.tanh(y)
            x = oracle.bf16_round(y)
        if kind == "port":
            secs = time.perf_counter() - t0
        return secs, nimg, kind

    def parity(self):
        """Sampled images of the timed output against the oracle chain (bf16
        rounding between layers, ReLU / tanh as fused), reference
        tensors_equal_approx form (tensor.hpp:275-286), tol 1e-2 (bf16 path)."""
        import oracle
        b = self.hi - self.lo
        idx = sorted({0, max(0, b // 2 - 1), b - 1})
        got = self.stack.out[idx].float().cpu().numpy()
        h = oracle.bf16_round(self.x_host[idx])
        for s, k in zip(self.specs, self.k_host):
            h = oracle.tconv_fused(h, oracle.bf16_round(k), s.p)
            h = oracle.bf16_round(np.maximum(h, 0) if s.activation == "relu" else np.tanh(h))
        return {"max_scaled_err": scaled_err(got, h), "tol": 1e-2,
                "images": [self.lo + i for i in idx], "oracle": "oracle.tconv_fused chain (C port, pinned)"}


def scaled_err(got, want):
    """max |a - b| / max(|a|, |b|, 1) -- the reference's tensors_equal_approx measure."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    if got.shape != want.shape:
        return float("inf")
    if got.size == 0:
        return 0.0
    return float((np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)).max())


def stack_specs(cfg):
    """Layer chain of a stack config: BASELINE C5, or a GAN generator preset."""
    from paper_2209_03704_b200 import stack as st
    return st.gan_layers(cfg["gan"]) if cfg.get("gan") else st.c5_layers()


def stack_macs_per_image(cfg):
    from oracle.oracle import count_ops
    return sum(count_ops(s.n_in, s.cin, s.cout, s.k, s.k, s.p)[2] for s in stack_specs(cfg))




def config_dict(name, cfg, world, bwd=False):
    """The `config` object of BOTH arms (identical, so the driver's same-config
    check holds): the workload and how the batch is split, nothing arm-specific."""
    batch = cfg["batch"]
    return {"workload": f"{name}: {cfg['desc']}" + (" -- backward (input + kernel gradients)" if bwd else ""),
            "global_batch": batch if cfg.get("stack") else batch * world,
            "per_rank_batch": (batch + world - 1) // world if cfg.get("stack") else batch,
            "parallelism": f"batch-sharded x{world}, weights replicated"
            + (" (all-gather of the outputs reported as gather_ms)" if cfg.get("stack") else "")
            + (", kernel-gradient all-reduce overlapped with the input gradient" if bwd and world > 1 else ""),
            "l2": "GPU arm: flushed between timed steps (256 MiB write outside the events); "
                  "CPU arm: not applicable"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """`--gpus N` without an outer launcher: re-run this script as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1).  NCCL
    init logging stays on (on stderr, so stdout keeps one JSON line)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    log("bench: launching", args.gpus, "ranks:", " ".join(cmd))
    sys.exit(subprocess.run(cmd, env=env).returncode)


# ------------------------------------------------------------ reference arm
def run_reference(args, cfg, world):
    """`--impl reference`: the reference's own CPU implementation (oracle/_ref, built
    from the unmodified headers) on this box's host cores, same metric/config.
    Value: images spread over all host threads, each through the reference's
    sequential transpose_conv_fused (the fastest way to run it on this host);
    the reference's own threaded transpose_conv_fused_parallel is reported beside it."""
    import oracle
    workers = os.cpu_count() or 1
    kind = "reference" if oracle.ref_available() else "port"
    name = args.config
    rng = np.random.default_rng(SEED)
    times, par_times = [], []
    extra_times = {}  # sequential op, conventional naive path: (seconds, images)
    bwd = args.pass_ == "backward"
    if cfg.get("stack"):
        specs = stack_specs(cfg)
        krng = np.random.default_rng(SEED)
        ks = [oracle.bf16_round(gen((s.k, s.k, s.cin, s.cout), "n02", krng)) for s in specs]
        nimg = min(cfg["batch"], max(1, 2 * workers))
        s0 = specs[0]
        x0 = oracle.bf16_round(rng.standard_normal((nimg, s0.n_in, s0.n_in, s0.cin), dtype=np.float32))
        macs = stack_macs_per_image(cfg) * nimg

        def chain(mode, w, n):
            x, secs = x0[:n], 0.0
            for s, k in zip(specs, ks):
                if kind == "reference":
                    y, dt = oracle.ref_time_fused_batch(mode, x, k, s.p, w)
                else:
                    t0 = time.perf_counter()
                    y = oracle.tconv_fused(x, k, s.p)
                    dt = time.perf_counter() - t0
                secs += dt
                x = oracle.bf16_round(np.maximum(y, 0) if s.activation == "relu" else np.tanh(y))
            return secs
        for i in range(args.warmup + args.steps):
            secs = chain(1, workers, nimg)
            if i >= args.warmup:
                times.append(secs)
        if kind == "reference":  # the reference's own threading, a bounded sample
            npar = min(nimg, 4)
            par_times.append((chain(0, workers, npar), npar))
            extra_times["sequential"] = (chain(1, 1, 1), 1)
            extra_times["naive"] = (chain(2, workers, min(nimg, workers)), min(nimg, workers))
    else:
        b, n, cin, cout, k, p = (cfg[x] for x in ("batch", "n", "cin", "cout", "k", "p"))
        nimg = min(b, max(1, 2 * workers))
        x = gen((nimg, n, n, cin), cfg["xd"], rng)
        kk = gen((k, k, cin, cout), cfg["wd"], np.random.default_rng(SEED), fan_in=cin * k * k)
        if cfg["dtype"] == "bf16":
            x, kk = oracle.bf16_round(x), oracle.bf16_round(kk)
        from oracle.oracle import count_ops
        macs = count_ops(n, cin, cout, k, k, p)[2] * nimg
        if bwd:  # backward: 2x the forward's useful MACs; output gradient ~ N(0, 1)
            macs *= 2
            g = oracle.geometry(n, k, k, p)
            gy = rng.standard_normal((nimg, g.out_h, g.out_w, cout), dtype=np.float32)
            if cfg["dtype"] == "bf16":
                gy = oracle.bf16_round(gy)
        for i in range(args.warmup + args.steps):
            if kind == "reference":
                if bwd:
                    _, _, secs = oracle.ref_time_backward(x, kk, p, gy, workers)
                else:
                    _, secs = oracle.ref_time_fused_batch(1, x, kk, p, workers)
            else:
                t0 = time.perf_counter()
                if bwd:
                    oracle.tconv_backward(x, kk, p, gy)
                else:
                    oracle.tconv_fused(x, kk, p)
                secs = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(secs)
        if kind == "reference" and not bwd:
            npar = min(nimg, 4)
            _, secs = oracle.ref_time_fused_batch(0, x[:npar], kk, p, workers)
            par_times.append((secs, npar))
            _, secs = oracle.ref_time_fused_batch(1, x[:1], kk, p, 1)
            extra_times["sequential"] = (secs, 1)
            nn = min(nimg, workers)
            _, secs = oracle.ref_time_fused_batch(2, x[:nn], kk, p, workers)
            extra_times["naive"] = (secs, nn)
    sec = statistics.median(times)
    val = macs / sec / 1e9
    sample = (f"{nimg} of {cfg['batch']} images per step, harness batch-threading over the "
              f"reference's sequential transpose_conv_fused (images across {workers} threads)"
              if kind == "reference" else f"{nimg} images per step, single-thread C port")
    if bwd:
        sample = sample.replace("transpose_conv_fused",
                                "net::FusedTConv::backward (timed; its forward untimed)")
    cpu = {"value": round(val, 4), "unit": "useful GMAC/s",
           "cores": workers if kind == "reference" else 1, "kind": kind, "sample": sample,
           "cpu_model": cpu_model()}
    if par_times:
        secs, npar = par_times[0]
        cpu["reference_parallel"] = {
            "value": round(macs / nimg * npar / secs / 1e9, 4), "unit": "useful GMAC/s",
            "what": f"the reference's own transpose_conv_fused_parallel({workers} workers; threads over "
                    f"cout slices, capped at cout) per image, {npar} images"}
    if "sequential" in extra_times:
        secs, ni = extra_times["sequential"]
        cpu["reference_sequential"] = {
            "value": round(macs / nimg * ni / secs / 1e9, 4), "unit": "useful GMAC/s",
            "what": "the reference's sequential transpose_conv_fused on one thread, 1 image"}
    if "naive" in extra_times:
        secs, ni = extra_times["naive"]
        cpu["reference_naive"] = {
            "value": round(macs / nimg * ni / secs / 1e9, 4), "unit": "useful GMAC/s (the fused op's MACs)",
            "what": f"the conventional transpose_conv_naive (upsample + pad + valid conv, 4x the MACs), "
                    f"{ni} images across {workers} threads"}
    out = {"metric": METRIC + (" [backward pass]" if bwd else ""),
           "value": round(val, 4), "unit": "useful GMAC/s", "impl": "reference",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
           "scaling": "strong" if cfg.get("stack") else "weak", "vs_baseline": None,
           "dtype": "f32", "data": "synthetic (seeded, BASELINE distributions; no dataset)",
           "config": config_dict(name, cfg, world, bwd),
           "cpu_baseline": cpu,
           "e2e": {"value": round(val, 4), "unit": "useful GMAC/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------- launcher check (CPU, gloo)
def run_plumbing_check(args, cfg, world, rank):
    """`--plumbing-check`: the multi-rank plumbing of the GPU arm on CPU (gloo):
    rendezvous, batch shards, the weight broadcast, max-over-ranks timing
    reduction and the output all-gather -- no convolution is computed.  Used by
    the CPU test of `--gpus N` self-launch; never a bench number."""
    import torch
    import torch.distributed as dist
    from paper_2209_03704_b200 import stack as st
    if world > 1:
        dist.init_process_group("gloo")
    b = cfg["batch"]
    lo, hi = st.shard_range(b, rank, world)
    w = torch.arange(16, dtype=torch.float32) if rank == 0 else torch.zeros(16)
    if world > 1:
        dist.broadcast(w, src=0)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    local = torch.arange(lo, hi, dtype=torch.float32).reshape(-1, 1).repeat(1, 3)
    full = st.gather_shards(local, b) if world > 1 else local
    ok = bool(torch.equal(full[:, 0], torch.arange(b, dtype=torch.float32))) and bool(
        torch.equal(w, torch.arange(16, dtype=torch.float32)))
    if rank == 0:
        print(json.dumps({"plumbing_only": True, "n_gpus": world, "ranks_seen_max": float(t.item()),
                          "shard": [lo, hi], "gathered_rows": int(full.shape[0]), "ok": ok,
                          "config": config_dict(args.config, cfg, world)}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if not ok:
        sys.exit(1)


# ---------------------------------------------------------------- main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=os.environ.get("SEGCONV_BENCH_CONFIG", "C5"),
                    choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="segconv", choices=["segconv", "reference"])
    ap.add_argument("--no-baselines", action="store_true", help="skip conventional/cuDNN/CPU legs")
    ap.add_argument("--pass", dest="pass_", default="forward", choices=["forward", "backward"],
                    help="backward: the layer's input + kernel gradients (not for the C5 stack)")
    ap.add_argument("--no-e2e", action="store_true",
                    help="diagnostics (ncu launch lists): skip the host-buffer e2e leg")
    ap.add_argument("--no-parity", action="store_true", help="skip the sampled oracle check")
    ap.add_argument("--dist", action="store_true",
                    help="use the NCCL process group even at world size 1 (launcher plumbing check)")
    ap.add_argument("--batch", type=int, default=None,
                    help="diagnostics: override the config's batch (not a headline line)")
    ap.add_argument("--plumbing-check", action="store_true",
                    help="CPU (gloo) check of the multi-rank launch/shard/gather plumbing; no compute")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.batch is not None:
        cfg = dict(cfg, batch=args.batch, desc=cfg["desc"] + f" [batch overridden: {args.batch}]")

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}; reporting n_gpus = {world}")

    if args.plumbing_check:
        run_plumbing_check(args, cfg, world, rank)
        return
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg, world)
        return

    import torch
    import torch.distributed as dist

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the segconv arm has no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _DIST[0] = world > 1 or args.dist
    if dist_on():
        dist.init_process_group("nccl", device_id=dev)
    from paper_2209_03704_b200 import segconv as sc

    bwd = args.pass_ == "backward"
    if bwd and cfg.get("stack"):
        raise SystemExit("--pass backward runs on single-layer configs (C1-C4, C5a-d)")
    prob = Stack(cfg, rank, world, torch, sc, dev) if cfg.get("stack") else \
        (LayerBackward if bwd else Layer)(cfg, rank, torch, sc, dev, world)
    flush_buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.fill_(1)

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        flush()
        prob.step()
    torch.cuda.synchronize()
    # The timed step replays a CUDA graph of the hot path so host launch
    # overhead (ctypes, argument checks) is not on the device clock; the e2e
    # leg below goes through the public API eagerly.  (The stack captures its
    # own graph; the backward pass allocates its split-K workspace per call.)
    graph = None
    if not cfg.get("stack") and not bwd:
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            prob.step()
        stream.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            prob.step()
        torch.cuda.synchronize()
    run_step = graph.replay if graph is not None else prob.step
    for _ in range(2):
        flush()
        run_step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, each bracketed by events; L2 flushed between steps
    if dist_on():
        dist.barrier()
    torch.cuda.synchronize()
    l0 = sc.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with Clocks(local) as clk:
        for a, b in evs:
            flush()
            a.record(stream)
            run_step()
            b.record(stream)
        torch.cuda.synchronize()
    launches = sc.launch_count() - l0
    if graph is not None or cfg.get("stack"):
        # graph replays bypass the host-side counter: count the captured kernels
        launches = args.steps * prob.launches_per_step
    if dist_on():
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot_ms = sum(step_ms)
    t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
    if dist_on():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms = float(t.item())
    ms = tot_ms / args.steps
    macs_all = prob.macs * world if not cfg.get("stack") else prob.macs
    if cfg.get("stack") and dist_on():
        mt = torch.tensor([prob.macs], device=dev, dtype=torch.float64)
        dist.all_reduce(mt)
        macs_all = float(mt.item())
    value = macs_all / (ms * 1e-3) / 1e9

    # ---- parity of the timed output (sampled images vs the oracle), every rank
    parity = None
    if not args.no_parity:
        try:
            parity = prob.parity()
            parity["pass"] = bool(parity["max_scaled_err"] <= parity["tol"])
        except Exception as e:  # report, do not hide
            parity = {"error": str(e)[:200], "pass": False}
        if dist_on():
            pf = torch.tensor([0.0 if parity.get("pass") else 1.0], device=dev)
            dist.all_reduce(pf, op=dist.ReduceOp.MAX)
            parity["all_ranks_pass"] = bool(pf.item() == 0.0)

    # ---- the stack's exchange step: all-gather of the output shards, max over ranks
    gather = None
    if cfg.get("stack"):
        gms = 0.0
        if dist_on():
            for _ in range(2):
                prob.gather()
            torch.cuda.synchronize()
            dist.barrier()
            ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ga.record(stream)
            for _ in range(args.steps):
                full = prob.gather()
            gb.record(stream)
            torch.cuda.synchronize()
            gt = torch.tensor([ga.elapsed_time(gb) / args.steps], device=dev, dtype=torch.float64)
            dist.all_reduce(gt, op=dist.ReduceOp.MAX)
            gms = float(gt.item())
            assert full.shape[0] == prob.global_batch
        gather = {"ms": round(gms, 5), "bytes_total": int(prob.global_batch * prob.stack.out[0].numel() * 2),
                  "what": "ShardedStack.gather: NCCL all-gather of the bf16 output shards"
                          if dist_on() else "single rank: nothing to gather"}

    # ---- e2e through the public API with host buffers (H2D + compute + D2H)
    e2e_steps = 0 if args.no_e2e else args.steps
    for _ in range(2 if e2e_steps else 0):
        prob.step_e2e()
    torch.cuda.synchronize()
    if dist_on():
        dist.barrier()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    ea.record(stream)
    for _ in range(e2e_steps):
        prob.step_e2e()
    eb.record(stream)
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - w0) * 1e3
    # the C ABI stack driver runs on its own streams and returns when its
    # output is on the host: time it by the host clock (it is synchronous)
    per = (wall_ms if getattr(prob, "capi", None) is not None else ea.elapsed_time(eb)) / max(1, e2e_steps)
    e2e_ms = torch.tensor([per], device=dev, dtype=torch.float64)
    if dist_on():
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    h2d, d2h = prob.e2e_bytes()

    # ---- roofline of the dominant kernel: the single layer's kernel, or for the
    # stack the slowest of its per-layer kernels (timed per layer with events)
    pk = peaks()
    kern_ms = statistics.mean(step_ms)
    layers = None
    if cfg.get("stack"):
        layers = prob.layer_times(max(5, min(args.steps, 20)), flush)
        dom = max(layers, key=lambda l: l["ms"])
        roof = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                "frac": dom["frac"], "kernel": f"layer {dom['layer']} ({dom['path']})",
                "per_launch_ms": dom["ms"],
                "peak_src": pk["src"] + (" bf16 burst" if dom["bound"] == "tensor" else " copy")}
        ach = 2.0 * prob.macs / (kern_ms * 1e-3) / 1e12
        stack_roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": pk["bf16"], "unit": "TFLOP/s",
                      "frac": round(ach / pk["bf16"], 4),
                      "what": "whole step (4 layers, one graph, PDL between layers)"}
    elif prob.bound == "tensor":
        ach = 2.0 * prob.macs / (kern_ms * 1e-3) / 1e12
        div = getattr(prob, "tensor_peak_div", 1.0)
        roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": round(pk["bf16"] / div, 1),
                "unit": "TFLOP/s", "frac": round(ach * div / pk["bf16"], 4),
                "peak_src": pk["src"] + " bf16 burst" + (" / 3 (split-fp16: 3 MMAs per product)"
                                                          if div != 1.0 else "")}
    else:
        ach = prob.alg_bytes / (kern_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm"], "unit": "GB/s",
                "frac": round(ach / pk["hbm"], 4), "peak_src": pk["src"] + " copy"}
    roof["traffic"] = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        tr = json.load(open(prof)).get(args.config + (":backward" if bwd else ""))
        if tr:
            roof["traffic"] = tr.get("dram_bytes_per_launch")
            roof["traffic_src"] = tr.get("source")
    hbm_gbs = prob.alg_bytes / (kern_ms * 1e-3) / 1e9

    # ---- strong-scaling proxy on one GPU: the per-GPU share of the global batch
    sweep = None
    if cfg.get("stack") and world == 1 and not args.no_baselines:
        sweep = {str(prob.global_batch): {"ms": round(ms, 5), "gmacs": round(value, 1)}}
        for share in (2, 4, 8):
            bb = prob.global_batch // share
            sub = Stack(cfg, 0, 1, torch, sc, dev, batch=bb, with_capi=False)
            for _ in range(3):
                flush()
                sub.step()
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.steps):
                flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                sub.step()
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            sms = statistics.mean(ts)
            sweep[str(bb)] = {"ms": round(sms, 5), "gmacs": round(sub.macs / (sms * 1e-3) / 1e9, 1),
                              "projected_n_gpus": share,
                              "projected_value": round(prob.macs / (sms * 1e-3) / 1e9, 1)}
            del sub
        sweep["note"] = ("one GPU timing the per-GPU batch of the 1/2/4/8-GPU split (projected_value = "
                         "the global batch's MACs over that time, gather excluded)")

    out = None
    if rank == 0:
        extra = {}
        if not args.no_baselines and world == 1:
            try:
                extra["conventional_gpu"] = prob.conventional(torch, 5, flush)
            except Exception as e:  # report, do not hide
                extra["conventional_gpu"] = {"error": str(e)[:200]}
            # cuDNN context.  fp32 data: strict fp32 (allow_tf32 off, the like-for-like
            # number at our 1e-5 bar) and torch's default TF32 (10-bit mantissa) both.
            fp32 = getattr(prob, "tdt", None) == torch.float32
            for tf32, key in ((False, "cudnn_conv_transpose2d"), (True, "cudnn_conv_transpose2d_tf32")):
                if tf32 and not fp32:
                    continue
                prev = torch.backends.cudnn.allow_tf32
                torch.backends.cudnn.allow_tf32 = tf32
                try:
                    r = prob.cudnn(torch, 5, flush)
                    if r and fp32:
                        r["what"] += " [TF32 math]" if tf32 else " [strict fp32: allow_tf32=False]"
                    extra[key] = r
                except Exception as e:
                    extra[key] = {"error": str(e)[:200]}
                finally:
                    torch.backends.cudnn.allow_tf32 = prev
            if bwd:
                extra["cudnn_conv_transpose2d_backward"] = extra.pop("cudnn_conv_transpose2d")
                if "cudnn_conv_transpose2d_tf32" in extra:
                    extra["cudnn_conv_transpose2d_backward_tf32"] = extra.pop("cudnn_conv_transpose2d_tf32")
                if fp32:
                    try:
                        extra["f16x3_backward"] = prob.f16x3_leg(torch, 10, flush)
                    except Exception as e:
                        extra["f16x3_backward"] = {"error": str(e)[:200]}
            workers = os.cpu_count() or 1
            try:
                secs, nimg, kind = prob.cpu_sample(workers)
                per_img = prob.macs / (cfg["batch"] if not cfg.get("stack") else prob.stack.batch)
                cpu_val = per_img * nimg / secs / 1e9
                extra["cpu_baseline"] = {
                    "value": round(cpu_val, 4), "unit": "useful GMAC/s",
                    "cores": workers if kind == "reference" else 1, "kind": kind,
                    "cpu_model": cpu_model(),
                    "sample": (f"{nimg} images of the same workload, reference "
                               + ("net::FusedTConv::backward (timed; its forward untimed)" if bwd
                                  else "transpose_conv_fused")
                               + f" per image, images across {workers} host threads, one pass")}
            except Exception as e:
                extra["cpu_baseline"] = {"error": str(e)[:200]}
        out = {"metric": METRIC + (" [backward pass]" if bwd else ""), "value": round(value, 2),
               "unit": "useful GMAC/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": round(ms, 5), "higher_is_better": True,
               "scaling": "strong" if cfg.get("stack") else "weak", "vs_baseline": None,
               "dtype": "bf16" if cfg["dtype"] == "bf16" else "f32",
               "data": "synthetic (seeded, BASELINE distributions; no dataset)",
               "config": config_dict(args.config, cfg, world, bwd),
               "math": prob.math,
               "hbm_gbs": round(hbm_gbs, 1),
               "roofline": roof,
               "e2e": None if not e2e_steps else {
                       "value": round(macs_all / (e2e_ms * 1e-3) / 1e9, 2), "unit": "useful GMAC/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "ms_per_step": round(e2e_ms, 4),
                       "what": getattr(prob, "e2e_what", "C ABI segconv_transpose_conv_fused_host (pinned host "
                                       "buffers, batch slices pipelined over H2D / kernel / D2H streams)"),
                       **({"phases_ms": prob.capi.last_timing} if getattr(prob, "capi", None) is not None
                          else {})},  # None: --no-e2e (diagnostic runs only)
               "gpu_launches": int(launches),
               "parity": parity,
               "clocks": clk.summary()}
        if cfg.get("stack"):
            out["stack_roofline"] = stack_roof
            out["layers"] = layers
            out["gather_ms"] = gather
            if sweep:
                out["strong_scaling_proxy"] = sweep
        out.update(extra)
        print(json.dumps(out), flush=True)
    if dist_on():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
