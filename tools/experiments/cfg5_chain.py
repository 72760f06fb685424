"""Config-5 chain ttv -> ttm -> norm from a cold L2 (CUDA-graph difference
against 512 MB read flushes, as bench.py's cold()), per seeded layout, under
the environment's knobs (e.g. TL_TTV_KEEP_MB)."""
import os, sys, json, statistics
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import torch
import paper_1711_10912_b200 as tl
from paper_1711_10912_b200 import contraction as C
import workloads as W
flush_buf = torch.ones((512 << 20) // 4, dtype=torch.float32, device="cuda")
sink = torch.empty(1, dtype=torch.float32, device="cuda")

def cold(fn, reps=20, iters=5):
    fn(); fn(); torch.cuda.synchronize()
    gs = []
    for with_fn in (True, False):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                torch.sum(flush_buf, dim=0, keepdim=True, out=sink)
                if with_fn:
                    fn()
        gs.append(g)
    ts = {True: [], False: []}
    for _ in range(iters):
        for with_fn, g in zip((True, False), gs):
            g.replay(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b.record(); torch.cuda.synchronize()
            ts[with_fn].append(a.elapsed_time(b))
    return (statistics.median(ts[True]) - statistics.median(ts[False])) / reps * 1e3

out = {"keep_mb": os.environ.get("TL_TTV_KEEP_MB", "128")}
for seed in (0, 5):
    T, v, M, layout = W.cfg5(seed)
    A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, layout), layout=layout)
    del T
    Vv = tl.DenseTensor.from_memory((9,), v)
    Bm = tl.DenseTensor.from_memory(M.shape, W.layout_buffer(M, (1, 2)))
    def chain():
        return C.frobenius_norm_device(tl.ttm(tl.ttv(A, Vv, 5), Bm, 2))
    def ttv_only():
        return tl.ttv(A, Vv, 5)
    out[f"seed{seed}_chain_us"] = round(cold(chain), 1)
    out[f"seed{seed}_ttv_us"] = round(cold(ttv_only), 1)
    out[f"seed{seed}_norm"] = float(chain().item())
    del A
    torch.cuda.empty_cache()
print(json.dumps(out))
