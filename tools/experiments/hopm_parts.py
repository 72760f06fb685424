"""Config-4 HOPM: one sweep's time against its parts timed alone (graph replays)."""
import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests")); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
import workloads as W
from sweep_ttm5 import timeit
T, _ = W.cfg4()
A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3)))
del T
u = tl.DenseTensor.from_memory((400,), np.full(400, 400 ** -0.5))
out = {}
out["pass_mode3_us"] = round(timeit(lambda: tl.ttv(A, u, 3), n=10), 2)
out["pass_mode2_us"] = round(timeit(lambda: tl.ttv(A, u, 2), n=10), 2)
P = tl.ttv(A, u, 3)
out["fold_400x400_k2_us"] = round(timeit(lambda: tl.ttv(P, u, 2)), 2)
out["fold_400x400_k1_us"] = round(timeit(lambda: tl.ttv(P, u, 1)), 2)
r = tl.HopmRunner(A, max_sweeps=50, tol=0.0)
r.launch(); torch.cuda.synchronize()
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); r.launch(); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
out["sweep_us"] = round(min(ts) * 1e3 / 50, 2)
print(json.dumps(out))
