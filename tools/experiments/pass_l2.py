"""How much does a HOPM pass over A (400^3 f64) gain when the rows it reads
first are already in L2?  Graph-difference timing: [flush, touch, pass] -
[flush, touch], touch = a read of the pass's first-read rows (mode 3: the
first k-planes; mode 2: the first rows of every o-slab)."""
import json
import statistics
import sys

import torch

sys.path[:0] = [".", "tests"]
import paper_1711_10912_b200 as tl  # noqa: E402
import workloads as W  # noqa: E402

T, _ = W.cfg4()
A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3)))
del T
u = tl.DenseTensor.from_memory((400,), [400 ** -0.5] * 400)
flush = torch.empty(256 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
buf = A.buffer


def touch_fn(mode, mb):
    if mb == 0:
        return lambda: None
    n = 400
    if mode == 3:
        nk = int(mb * 2 ** 20 / (n * n * 8))
        region = buf[: nk * n * n]
        return lambda: sink.copy_(region.sum().reshape(1))
    nk = int(mb * 2 ** 20 / (n * n * 8))  # rows per slab
    view = buf.view(n, n, n)[:, :nk, :]  # [o][k][i]
    return lambda: sink.copy_(view.sum().reshape(1))


def graph_time(fns, reps=10, iters=5):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fns:
            f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for r in range(reps):
            for f in fns:
                f()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    return statistics.median(ts)


res = {}
for mode in (3, 2):
    for mb in (0, 24, 48, 96):
        t = touch_fn(mode, mb)
        fl = lambda: flush.fill_(1.0)  # noqa: E731
        with_pass = graph_time([fl, t, lambda: tl.ttv(A, u, mode)])
        without = graph_time([fl, t])
        res[f"mode{mode}_{mb}MB"] = round(with_pass - without, 2)
print(json.dumps(res))
