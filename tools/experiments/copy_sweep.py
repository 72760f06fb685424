"""Relayout/transpose of the 1 GiB config-2 tensor: device time per call
(graph replays; 2 GiB of traffic each, inputs 8x L2)."""
import json
import statistics
import sys

import torch

sys.path[:0] = [".", "tests"]
import paper_1711_10912_b200 as tl  # noqa: E402
import workloads as W  # noqa: E402

T, _, _ = W.cfg2()
A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3, 4)))
del T


def med(fn, reps=5, iters=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
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
for tau in ((4, 3, 2, 1), (3, 1, 2, 4), (2, 1, 3, 4), (1, 3, 2, 4)):
    res[str(tau)] = round(med(lambda: tl.transpose(A, tau)), 1)
print(json.dumps(res))
