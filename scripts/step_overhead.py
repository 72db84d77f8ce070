"""Diagnostics: what a bench.py step costs besides the hot kernel -- an empty
event pair after the L2 flush, a one-kernel graph, the C2 graph with / without
the flush.  python scripts/step_overhead.py"""
import statistics, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2209_03704_b200 import segconv as sc
cfg = bench.CONFIGS["C2"]
prob = bench.Layer(cfg, 0, torch, sc, torch.device("cuda", 0), 1)
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
small = torch.empty(1024, device="cuda")
for _ in range(3): prob.step()
torch.cuda.synchronize()
def graph_of(fn):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): fn()
    torch.cuda.synchronize()
    return g
def timeit(run, pre):
    ts = []
    for i in range(30):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); b.synchronize()
        if i >= 5: ts.append(a.elapsed_time(b) * 1000)
    return statistics.median(ts)
g_hot = graph_of(prob.step)
g_small = graph_of(lambda: small.fill_(1.0))
print("empty (flush before)", timeit(lambda: None, lambda: flush.fill_(1)))
print("small kernel graph (flush before)", timeit(g_small.replay, lambda: flush.fill_(1)))
print("hot graph (flush before)", timeit(g_hot.replay, lambda: flush.fill_(1)))
print("hot graph (no flush)", timeit(g_hot.replay, lambda: None))
print("hot graph (small kernel before)", timeit(g_hot.replay, lambda: small.fill_(2.0)))
