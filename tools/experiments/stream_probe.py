"""Run the stream-kernel ttm shapes one by one (eager, synchronised) and report each."""
import os, sys, time
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
rng = np.random.default_rng(1)
for shape, J in [((3, 33, 5, 17, 2, 640), 16), ((5, 37, 20001), 7), ((5, 37, 20001), 16), ((5, 37, 20001), 24)]:
    X = tl.DenseTensor.from_memory(shape, rng.standard_normal(shape).reshape(-1, order="F"))
    M = tl.DenseTensor.from_memory((J, shape[1]), rng.standard_normal((J, shape[1])).reshape(-1, order="F"))
    t = time.time()
    C = tl.ttm(X, M, 2)
    torch.cuda.synchronize()
    print(shape, J, "ok", round(time.time() - t, 3), flush=True)
shape, J = (3, 33, 5, 17, 2, 640), 16
X = tl.DenseTensor.from_memory(shape, rng.standard_normal(shape).reshape(-1, order="F"))
M = tl.DenseTensor.from_memory((J, shape[1]), rng.standard_normal((J, shape[1])).reshape(-1, order="F"))
ref = tl.ttm(X, M, 2).numpy()
for n in (2, 5, 20, 100):
    t = time.time()
    outs = [tl.ttm(X, M, 2) for _ in range(n)]
    torch.cuda.synchronize()
    bad = sum(int(not np.array_equal(o.numpy(), ref)) for o in outs)
    print("eager x", n, "ok", round(time.time() - t, 3), "mismatches", bad, flush=True)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    tl.ttm(X, M, 2)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
print("side stream ok", flush=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    outs = [tl.ttm(X, M, 2) for _ in range(20)]
print("captured", flush=True)
g.replay(); torch.cuda.synchronize()
print("replayed", sum(int(not np.array_equal(o.numpy(), ref)) for o in outs), flush=True)
