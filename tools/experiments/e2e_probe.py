import os, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch, numpy as np
import bench
wl = bench.Cfg2Workload()
first_buf, first_layout = wl.host["first"]
wl.pinned = {"first": (torch.from_numpy(first_buf).pin_memory(), first_layout)}
wl.pinned_T2 = torch.from_numpy(wl.host_T2).pin_memory()
wl.pinned_vecs = [torch.from_numpy(v).pin_memory() for v in wl.host_vecs]
wl.side_stream = torch.cuda.Stream()
print("pinned?", wl.pinned["first"][0].is_pinned(), wl.pinned_T2.is_pinned())
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); bench.e2e_step(wl); print("e2e step", time.perf_counter()-t)
x = wl.pinned["first"][0]
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); y = x.to("cuda", non_blocking=True); torch.cuda.synchronize(); print("h2d 1GB", time.perf_counter()-t)
import paper_1711_10912_b200 as tl
for i in range(2):
    torch.cuda.synchronize(); t=time.perf_counter(); A = tl.DenseTensor.from_memory(W.CFG2_SHAPE if False else (128,)*4, x, layout=(1,2,3,4)); torch.cuda.synchronize(); print("from_memory 1GB", time.perf_counter()-t)
