"""Batch-sharded multi-GPU driver logic on CPU with gloo (world size 2).

`ShardedStack` (paper_2209_03704_b200/stack.py) owns: the batch partition,
the one-time weight broadcast from rank 0 and the output all-gather.  The
per-rank compute (`GeneratorStack`, sm_100a kernels) is replaced here by a
CPU stand-in built on the oracle -- test infrastructure only -- so the
collective logic is exercised without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2209_03704_b200 import stack as st


def test_shard_range_partitions_batch():
    for batch in (1, 2, 7, 16, 1024, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [st.shard_range(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


class _CpuStack:
    """Stand-in for GeneratorStack: the same chain on the oracle, fp32."""

    def __init__(self, specs, kernels, batch, **kw):
        self.specs = list(specs)
        self.kernels = [k.detach().cpu().numpy().astype(np.float32) for k in kernels]
        self.batch = batch
        self.out = None

    def forward(self, x):
        h = x.numpy()
        for s, k in zip(self.specs, self.kernels):
            h = oracle.tconv_fused(h, k, s.p)
            h = np.maximum(h, 0) if s.activation == "relu" else np.tanh(h)
        self.out = torch.from_numpy(np.ascontiguousarray(h))
        return self.out


SPECS = [st.LayerSpec(8, 6, 4, 3, 0, "relu"), st.LayerSpec(6, 3, 5, 3, 0, "tanh")]


def _worker(rank, world, port, batch, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st.GeneratorStack = _CpuStack
        rng = np.random.default_rng(100 + rank)  # ranks start with DIFFERENT weights
        ks = [torch.from_numpy(rng.normal(0, 0.2, (s.k, s.k, s.cin, s.cout)).astype(np.float32))
              for s in SPECS]
        sh = st.ShardedStack(SPECS, ks, batch)
        xr = np.random.default_rng(7).normal(0, 1, (batch, 4, 4, 8)).astype(np.float32)
        sh.forward(torch.from_numpy(xr[sh.lo:sh.hi]))
        full = sh.gather()
        w0 = [k.numpy() for k in sh.kernels]
        q.put((rank, sh.lo, sh.hi, full.numpy(), w0))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("batch", [5, 8])
def test_sharded_stack_gloo_world2(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, full0, w0), (r1, lo1, hi1, full1, w1) = res
    assert (lo0, hi1) == (0, batch) and hi0 == lo1
    for a, b in zip(w0, w1):  # weights replicated from rank 0
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(full0, full1)  # every rank holds the full batch
    # equals the single-process chain on rank 0's weights
    xr = np.random.default_rng(7).normal(0, 1, (batch, 4, 4, 8)).astype(np.float32)
    h = xr
    for s, k in zip(SPECS, w0):
        h = oracle.tconv_fused(h, k, s.p)
        h = np.maximum(h, 0) if s.activation == "relu" else np.tanh(h)
    np.testing.assert_allclose(full0, h, rtol=0, atol=1e-6)


# ---- data-parallel backward: the kernel gradient is all-reduced over ranks
def _bwd_worker(rank, world, port, batch, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2209_03704_b200 import dp
        # CPU stand-ins for the per-rank sm_100a kernels (oracle: test infrastructure)
        dp._segregate = lambda k, p, m: None
        dp._local_forward = lambda x, sks, g, m: torch.from_numpy(
            oracle.tconv_fused(x.numpy(), KB, PB))
        dp._local_kernel_grad = lambda x, k, p, g, m: torch.from_numpy(
            oracle.tconv_backward(x.numpy(), k.numpy(), p, g.numpy())[1])
        dp._local_input_grad = lambda x, k, p, g, m: torch.from_numpy(
            oracle.tconv_backward(x.numpy(), k.numpy(), p, g.numpy())[0])
        rng = np.random.default_rng(300 + rank)  # different on each rank: rank 0's wins
        k = torch.from_numpy(rng.uniform(-1, 1, KB.shape).astype(np.float32))
        layer = dp.ShardedFusedTConv(k, PB, batch)
        x = np.random.default_rng(5).uniform(-1, 1, (batch, 5, 5, 3)).astype(np.float32)
        g = np.random.default_rng(6).uniform(-1, 1, (batch, 10, 10, 2)).astype(np.float32)
        layer.forward(torch.from_numpy(x[layer.lo:layer.hi]))
        gx = layer.backward(torch.from_numpy(g[layer.lo:layer.hi]))
        q.put((rank, layer.lo, layer.hi, gx.numpy(), layer.grad.numpy(), layer.kernel_.numpy()))
    finally:
        dist.destroy_process_group()


KB = np.random.default_rng(4).uniform(-1, 1, (4, 4, 3, 2)).astype(np.float32)
PB = 2


@pytest.mark.parametrize("batch", [3, 6])
def test_sharded_backward_gloo_world2(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bwd_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, lo0, hi0, gx0, gk0, k0), (_, lo1, hi1, gx1, gk1, k1) = res
    np.testing.assert_array_equal(k0, k1)  # kernel replicated from rank 0
    x = np.random.default_rng(5).uniform(-1, 1, (batch, 5, 5, 3)).astype(np.float32)
    g = np.random.default_rng(6).uniform(-1, 1, (batch, 10, 10, 2)).astype(np.float32)
    wx, wk = oracle.tconv_backward(x, k0, PB, g)
    np.testing.assert_array_equal(np.concatenate([gx0, gx1]), wx)  # input grads: per shard
    np.testing.assert_array_equal(gk0, gk1)  # every rank holds the all-reduced sum
    np.testing.assert_allclose(gk0, wk, rtol=0, atol=1e-5)  # == the full-batch kernel grad


def test_multi_gpu_stack_checks_the_chain_on_the_host():
    """segconv_stack_create validates the layer chain before touching a device
    (ShapeError like the reference's geometry checks), so it fails the same way
    with or without a GPU."""
    from paper_2209_03704_b200 import segconv as sc
    from paper_2209_03704_b200 import stack as st
    specs = [st.LayerSpec(64, 32, 4, 3), st.LayerSpec(31, 16, 5, 3)]  # 5x5x32 does not feed cin 31
    ks = [torch.zeros((3, 3, 64, 32)), torch.zeros((3, 3, 31, 16))]
    with pytest.raises(sc.ShapeError, match="does not feed"):
        st.MultiGPUStack(specs, ks, 4, act_dtype=torch.float32)
