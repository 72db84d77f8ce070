"""Data-parallel training of the fused layer over torch.distributed ranks.

The backward pass (reference netdemo/layers.hpp:171-211) shards by image like
the forward, but its kernel gradient is a sum over the whole batch: that sum is
the path's one real exchange step.  `ShardedFusedTConv` keeps a batch shard per
rank (one GPU each), broadcasts rank 0's kernel once, and in `backward`
launches the kernel gradient first, starts its all-reduce (NCCL on GPU)
asynchronously, and computes the input gradient while the reduction is in
flight -- the collective overlaps the tensor-core input-gradient kernel.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import segconv as sc
from .stack import shard_range


def _local_forward(x, sks, geom, math):
    return sc.transpose_conv_fused(x, sks, geom, math=math)


def _local_kernel_grad(x, kernel, p, g, math):
    _, gk = sc.transpose_conv_fused_backward(x, kernel, p, g, math=math, input_grad=False)
    return gk


def _local_input_grad(x, kernel, p, g, math):
    gx, _ = sc.transpose_conv_fused_backward(x, kernel, p, g, math=math, kernel_grad=False)
    return gx


def _segregate(kernel, p, math):
    return sc.segregate(kernel, p, math=math or "auto")


class ShardedFusedTConv:
    """net::FusedTConv over `world` ranks: rank r owns images
    shard_range(global_batch, r, world); grad (the kernel gradient) is the
    all-reduced sum over the global batch on every rank."""

    def __init__(self, kernel: torch.Tensor, p: int, global_batch: int, *, group=None,
                 src_rank: int = 0, math: Optional[str] = None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.global_batch = int(global_batch)
        self.lo, self.hi = shard_range(self.global_batch, self.rank, self.world)
        k = kernel.contiguous()
        dist.broadcast(k, src=src_rank, group=group)  # replicated weights, once
        self.kernel_ = k
        self.p_ = int(p)
        self.math = math
        acc_dt = torch.float64 if k.dtype == torch.float64 else torch.float32
        self.grad = torch.zeros(k.shape, dtype=acc_dt, device=k.device)
        self._x = None
        self.on_params_updated()

    def on_params_updated(self) -> None:
        self.sks_ = _segregate(self.kernel_, self.p_, self.math)

    def params(self):
        return [(self.kernel_, self.grad)]

    def zero_grads(self) -> None:
        self.grad.zero_()

    def forward(self, x_local: torch.Tensor) -> torch.Tensor:
        if x_local.shape[0] != self.hi - self.lo:
            raise sc.ContractError(f"rank {self.rank} owns {self.hi - self.lo} images, got "
                                   f"{x_local.shape[0]}")
        self._x = x_local
        self.geom_ = sc.tconv_geometry(int(x_local.shape[1]), int(self.kernel_.shape[0]),
                                       int(self.kernel_.shape[1]), self.p_)
        return _local_forward(x_local, self.sks_, self.geom_, self.math)

    def backward(self, g_local: torch.Tensor) -> torch.Tensor:
        if self._x is None:
            raise sc.StateError("fused_tconv: backward called before forward")
        gk = _local_kernel_grad(self._x, self.kernel_, self.p_, g_local, self.math)
        work = self.dist.all_reduce(gk, op=self.dist.ReduceOp.SUM, group=self.group,
                                    async_op=True)
        gx = _local_input_grad(self._x, self.kernel_, self.p_, g_local, self.math)  # overlaps
        work.wait()
        self.grad += gk
        return gx
