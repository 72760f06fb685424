"""Small launches of every kernel family for compute-sanitizer runs."""
import os, sys
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
import workloads as W
rng = np.random.default_rng(0)
def T(shape, layout, dt=np.float64):
    x = rng.uniform(-1, 1, size=shape).astype(dt)
    return tl.DenseTensor.from_memory(shape, W.layout_buffer(x, layout), layout=layout)
def V(n, dt=np.float64):
    return tl.DenseTensor.from_memory((n,), rng.uniform(-1, 1, n).astype(dt))
# ttv regimes: strided, staged, rows-tma (f32 I==1), box (permuted, K<=32), small rows/cols
A = T((64, 40, 300), (1, 2, 3), np.float32); tl.ttv(A, V(64, np.float32), 1); tl.ttv(A, V(40, np.float32), 2)
B = T((9, 37, 5, 11), (3, 1, 2, 4)); tl.ttv(B, V(37), 2); tl.ttv(B, V(9), 1)
Cx = T((3, 9, 5, 640), (4, 2, 1, 3)); tl.ttv(Cx, V(9), 2)
D = T((400, 400), (1, 2)); tl.ttv(D, V(400), 1); tl.ttv(D, V(400), 2)
# ttm: GETT (f64, f32), bulk, staged permuted, SIMT
G = T((48, 40, 36), (3, 2, 1)); M = tl.DenseTensor.from_memory((64, 40), rng.standard_normal(64 * 40))
tl.ttm(G, M, 2)
G32 = T((48, 40, 36), (1, 2, 3), np.float32); tl.ttm(G32, M.to(torch.float32), 2)
Bk = T((5, 37, 201), (1, 2, 3)); tl.ttm(Bk, tl.DenseTensor.from_memory((16, 37), rng.standard_normal(16 * 37)), 2)
St = T((40, 999), (1, 2)); tl.ttm(St, tl.DenseTensor.from_memory((20, 40), rng.standard_normal(20 * 40)), 1)  # stream, partial tile
Sp = T((20, 33, 7), (2, 1, 3)); tl.ttm(Sp, tl.DenseTensor.from_memory((8, 33), rng.standard_normal(8 * 33)), 2)
# reductions, copy, hopm
tl.inner_product_tensors(A, A); tl.frobenius_norm(B); tl.frobenius_norm(G)
Cx.relayout((1, 2, 3, 4))
st = tl.hopm(T((12, 10, 8), (1, 2, 3)), max_sweeps=3, tol=0.0)
torch.cuda.synchronize()
print("ok")
