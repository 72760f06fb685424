"""One 400x400 small ttv in each shape, then two HOPM sweeps on 400^3, inside a profiler window."""
import os, sys
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import torch
import paper_1711_10912_b200 as tl
import workloads as W
P = tl.DenseTensor.from_memory((400, 400), torch.randn(160000, dtype=torch.float64, device="cuda"))
v = tl.DenseTensor.from_memory((400,), torch.randn(400, dtype=torch.float64, device="cuda"))
T, _ = W.cfg4()
A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3)))
r = tl.HopmRunner(A, max_sweeps=2, tol=0.0)
for _ in range(2):
    tl.ttv(P, v, 1); tl.ttv(P, v, 2); r.launch()
torch.cuda.synchronize()
torch.cuda.profiler.start()
tl.ttv(P, v, 1); tl.ttv(P, v, 2); r.launch()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
