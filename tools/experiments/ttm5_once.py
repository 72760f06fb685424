"""One cfg5 ttm (16x33 matrix, mode 2 of the seed-0 ttv output) inside a
profiler window, for ncu cold timing sweeps (tools/experiments/ttm5_sweep.sh)."""
import sys

import torch

sys.path[:0] = [".", "tests"]
import paper_1711_10912_b200 as tl  # noqa: E402
import workloads as W  # noqa: E402

T, v, M, layout = W.cfg5(0)
A5 = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, layout), layout=layout)
del T
C1 = tl.ttv(A5, tl.DenseTensor.from_memory((9,), v), 5)
del A5
Bm = tl.DenseTensor.from_memory(M.shape, W.layout_buffer(M, (1, 2)))
for _ in range(2):
    tl.ttm(C1, Bm, 2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(3):
    tl.ttm(C1, Bm, 2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
