"""Multi-layer generator stack (BASELINE C5) and its batch-sharded driver.

A stack is a chain of segregated transpose convolutions, each output (2N-n)
feeding the next layer, ReLU fused into the epilogue of every layer but the
last, tanh fused into the last.  Activations stay in HBM in bf16 between
layers (the BASELINE's storage type) with fp32 accumulation inside each layer.

``GeneratorStack.forward`` launches one kernel per layer on the current
stream; ``capture()`` records the whole stack into a CUDA graph so a step is a
single graph launch (no per-layer host overhead).

Multi-GPU (``ShardedStack``): one process per GPU.  Rank 0's weights are
broadcast once with NCCL (``torch.distributed.broadcast``); each rank owns a
contiguous slice of the batch and runs the stack on it with no data-path
collective; ``gather`` all-gathers the output slices when the caller wants the
full batch.  There are no inter-layer exchanges.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from . import segconv as sc


@dataclass(frozen=True)
class LayerSpec:
    cin: int
    cout: int
    n_in: int
    k: int
    p: int = 0
    activation: Optional[str] = "relu"


def c5_layers() -> List[LayerSpec]:
    """BASELINE C5: 1024->512 N=4, 512->256 N=5, 256->128 N=7, 128->3 N=11, n=3."""
    return [LayerSpec(1024, 512, 4, 3, 0, "relu"), LayerSpec(512, 256, 5, 3, 0, "relu"),
            LayerSpec(256, 128, 7, 3, 0, "relu"), LayerSpec(128, 3, 11, 3, 0, "tanh")]


# reference proj/include/segconv/analysis.hpp:96-114 (gan_models): every
# transpose-conv layer of the named generator, 4x4 kernels at p = 2 (out = 2N);
# (layer index, N, cin, cout).  ReLU between layers, tanh on the last.
GAN_MODELS = {
    "dcgan": [(2, 4, 1024, 512), (3, 8, 512, 256), (4, 16, 256, 128), (5, 32, 128, 3)],
    "artgan": [(2, 4, 512, 256), (3, 8, 256, 128), (4, 16, 128, 128), (6, 32, 128, 3)],
    "gpgan": [(2, 4, 512, 256), (3, 8, 256, 128), (4, 16, 128, 64), (5, 32, 64, 3)],
    "ebgan": [(2, 4, 2048, 1024), (3, 8, 1024, 512), (4, 16, 512, 256), (5, 32, 256, 128),
              (6, 64, 128, 64), (7, 128, 64, 64)],
}


def gan_layers(model: str) -> List[LayerSpec]:
    """The generator's layers as a chain (reference analysis.hpp:96-121, gan_model)."""
    if model not in GAN_MODELS:
        raise sc.ContractError(f"unknown GAN model '{model}' (known: {', '.join(GAN_MODELS)})")
    rows = GAN_MODELS[model]
    return [LayerSpec(cin, cout, n, 4, 2, "tanh" if i == len(rows) - 1 else "relu")
            for i, (_, n, cin, cout) in enumerate(rows)]


def shard_range(batch: int, rank: int, world: int):
    """Contiguous batch slice [lo, hi) owned by `rank` (balanced, remainder first)."""
    base, rem = divmod(batch, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


class GeneratorStack:
    def __init__(self, specs: Sequence[LayerSpec], kernels: Sequence[torch.Tensor],
                 batch: int, *, act_dtype=torch.bfloat16, math: str = "auto",
                 biases: Optional[Sequence[Optional[torch.Tensor]]] = None):
        if len(specs) != len(kernels) or not specs:
            raise sc.ContractError("one kernel per layer spec is required")
        for a, b in zip(specs, specs[1:]):
            ga = sc.tconv_geometry(a.n_in, a.k, a.k, a.p)
            if ga.out_h != b.n_in or a.cout != b.cin:
                raise sc.ShapeError(f"layer output {ga.out_h}x{a.cout} does not feed "
                                    f"{b.n_in}x{b.cin}")
        self.specs = list(specs)
        self.batch = int(batch)
        self.act_dtype = act_dtype
        self.geoms = [sc.tconv_geometry(s.n_in, s.k, s.k, s.p) for s in specs]
        self.sks = [sc.segregate(k.to(act_dtype), s.p, math=math) for s, k in zip(specs, kernels)]
        self.biases = list(biases) if biases is not None else [None] * len(specs)
        dev = torch.device("cuda", torch.cuda.current_device())
        s0 = specs[0]
        self.x = torch.empty((batch, s0.n_in, s0.n_in, s0.cin), dtype=act_dtype, device=dev)
        self.acts = [torch.empty((batch, g.out_h, g.out_w, s.cout), dtype=act_dtype, device=dev)
                     for s, g in zip(specs, self.geoms)]
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    @property
    def out(self) -> torch.Tensor:
        return self.acts[-1]

    def useful_macs(self) -> int:
        return sum(sc.count_ops_fused(sc.LayerShape(s.n_in, s.cin, s.cout, s.k, s.k, s.p)).mults
                   for s in self.specs) * self.batch

    def algorithmic_bytes(self) -> int:
        """input + weights + output of every layer, each touched once (bf16)."""
        e = torch.tensor([], dtype=self.act_dtype).element_size()
        tot = 0
        for s, g in zip(self.specs, self.geoms):
            tot += (self.batch * s.n_in * s.n_in * s.cin + s.k * s.k * s.cin * s.cout +
                    self.batch * g.out_h * g.out_w * s.cout) * e
        return tot

    def _run(self):
        src = self.x
        for s, g, sks, dst, b in zip(self.specs, self.geoms, self.sks, self.acts, self.biases):
            sc.transpose_conv_fused(src, sks, g, bias=b, activation=s.activation, out=dst)
            src = dst

    def forward(self, x: Optional[torch.Tensor] = None) -> torch.Tensor:
        if x is not None:
            if tuple(x.shape) != tuple(self.x.shape):
                raise sc.ContractError(f"stack input must be {tuple(self.x.shape)}")
            self.x.copy_(x, non_blocking=True)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._run()
        return self.out

    def capture(self) -> None:
        """Record the layer chain into one CUDA graph (after one eager warm-up)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._run()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._run()
        self.graph = g


class ShardedStack:
    """Batch-sharded stack over torch.distributed ranks (one GPU each)."""

    def __init__(self, specs: Sequence[LayerSpec], kernels: Sequence[torch.Tensor],
                 global_batch: int, *, group=None, src_rank: int = 0, **kw):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.global_batch = int(global_batch)
        self.lo, self.hi = shard_range(global_batch, self.rank, self.world)
        ks = []
        for k in kernels:  # weights replicated: one broadcast from src_rank, once
            k = k.contiguous()
            dist.broadcast(k, src=src_rank, group=group)
            ks.append(k)
        self.kernels = ks
        self.local = GeneratorStack(specs, ks, self.hi - self.lo, **kw)

    def forward(self, x_local: Optional[torch.Tensor] = None) -> torch.Tensor:
        return self.local.forward(x_local)

    def gather(self) -> torch.Tensor:
        """All-gather the per-rank output slices into the full batch (every rank)."""
        return gather_shards(self.local.out, self.global_batch, group=self.group)


def gather_shards(local: torch.Tensor, global_batch: int, *, group=None) -> torch.Tensor:
    """The batch's per-rank slices (shard_range order) all-gathered into the full
    batch on every rank.  Uneven shards are padded to the largest one so a
    single all_gather moves them (NCCL over NVLink on GPU, gloo on CPU)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = local.contiguous()
    sizes = [shard_range(global_batch, r, world) for r in range(world)]
    maxb = max(h - l for l, h in sizes)
    if out.shape[0] == maxb:
        pad = out
    else:
        pad = out.new_zeros((maxb,) + tuple(out.shape[1:]))
        pad[: out.shape[0]].copy_(out)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: h - l] for b, (l, h) in zip(bufs, sizes)], dim=0)


class MultiGPUStack:
    """The C ABI's single-process multi-GPU driver (segconv_stack_*,
    csrc/stack.cu): one host thread, one stream per GPU, weights
    ncclBroadcast once at creation, each GPU a contiguous batch shard, the
    output shards ncclAllGather-ed; host tensors in, host tensor out.

    ``kernels`` are host (kh, kw, cin, cout) tensors; activations are
    ``act_dtype`` (bfloat16 or float32).  ``forward(x)`` takes a host
    (B, N, N, cin) tensor (page-locked for full-speed copies) and returns the
    host output plus the per-phase timing (max over GPUs)."""

    def __init__(self, specs: Sequence[LayerSpec], kernels: Sequence[torch.Tensor], max_batch: int, *,
                 n_gpus: int = 0, act_dtype=torch.bfloat16, biases=None):
        import ctypes as C
        from . import _capi as A
        if len(specs) != len(kernels) or not specs:
            raise sc.ContractError("one kernel per layer spec is required")
        self._A, self._C = A, C
        self.specs = list(specs)
        self.act_dtype = act_dtype
        self._keep = []
        arr = (A.Layer * len(specs))()
        for i, (s, k) in enumerate(zip(specs, kernels)):
            kh = k.detach().to("cpu").contiguous()
            self._keep.append(kh)
            b = None
            if biases is not None and biases[i] is not None:
                b = biases[i].detach().to("cpu", torch.float32).contiguous()
                self._keep.append(b)
            epi = sc._ACT[s.activation] | (A.EPI_BIAS if b is not None else 0)
            arr[i] = A.Layer(s.n_in, s.cin, s.cout, s.k, s.k, s.p, kh.data_ptr(), sc._DT[kh.dtype],
                             b.data_ptr() if b is not None else None, epi, A.MATH_AUTO)
        h = C.c_void_p()
        sc._check(A.lib().segconv_stack_create(arr, len(specs), sc._DT[act_dtype], int(max_batch), int(n_gpus),
                                               C.byref(h)))
        self._h = h
        self.n_gpus = int(A.lib().segconv_stack_gpus(h))
        g = sc.tconv_geometry(specs[-1].n_in, specs[-1].k, specs[-1].k, specs[-1].p)
        self.out_shape = (g.out_h, g.out_w, specs[-1].cout)
        self.last_timing = None

    def forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        A, C = self._A, self._C
        s0 = self.specs[0]
        if x.dim() != 4 or tuple(x.shape[1:]) != (s0.n_in, s0.n_in, s0.cin) or x.dtype != self.act_dtype:
            raise sc.ContractError(f"stack input must be (B, {s0.n_in}, {s0.n_in}, {s0.cin}) {self.act_dtype}")
        x = x.contiguous()
        if out is None:
            out = torch.empty((x.shape[0],) + self.out_shape, dtype=self.act_dtype)
        t = A.Timing()
        sc._check(A.lib().segconv_stack_forward(self._h, x.data_ptr(), int(x.shape[0]), out.data_ptr(),
                                                C.byref(t)))
        self.last_timing = {k: getattr(t, k) for k, _ in A.Timing._fields_}
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._A.lib().segconv_stack_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
