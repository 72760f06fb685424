"""Small launches of the few-row ttm kernels (csrc/ttm_few.cu: DMMA persistent boxes, SIMT boxes, every store
order, masked last boxes, float32 / int64), the 16/32-row GETT tiles, the reduced-row staged ttv and the
vectorised inner row walk, for compute-sanitizer (memcheck / racecheck) runs."""
import os, sys
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
import workloads as W
rng = np.random.default_rng(0)
def T(shape, layout, dt=np.float64):
    x = rng.integers(-9, 9, size=shape) if dt == np.int64 else rng.uniform(-1, 1, size=shape).astype(dt)
    return tl.DenseTensor.from_memory(shape, W.layout_buffer(x, layout), layout=layout)
def M(j, k, dt=np.float64):
    x = rng.integers(-9, 9, size=(j, k)) if dt == np.int64 else rng.standard_normal((j, k)).astype(dt)
    return tl.DenseTensor.from_memory((j, k), W.layout_buffer(x, (1, 2)))
shape = (3, 33, 5, 17, 2, 40)
for lay in [(4, 3, 6, 5, 1, 2), (3, 6, 5, 2, 4, 1), (1, 2, 3, 4, 5, 6)]:
    for dt in (np.float64, np.float32, np.int64):
        A = T(shape, lay, dt)
        for mode in range(1, 7):
            for J in (1, 7, 16, 25):
                tl.ttm(A, M(J, shape[mode - 1], dt), mode)
# long folds, few rows: GETT 16/32-row tiles
G = T((300, 20, 31), (2, 3, 1)); tl.ttm(G, M(16, 300), 1); tl.ttm(G, M(30, 300), 1)
# ttv rows of 2 / 6 elements (reduced-row staged tiles), slab scramble edge
V = lambda n: tl.DenseTensor.from_memory((n,), rng.uniform(-1, 1, n))
B = T((3, 33, 5, 17, 9, 2, 64), (6, 1, 2, 5, 3, 7, 4)); tl.ttv(B, V(3), 1); tl.ttv(B, V(64), 7); tl.ttv(B, V(33), 2)
B2 = T((3, 33, 5, 17, 9, 2, 64), (6, 7, 3, 4, 5, 1, 2)); tl.ttv(B2, V(64), 7)
# inner: shared fastest dimension, different outer order
a = T((64, 12, 10, 9), (1, 2, 3, 4)); b = T((64, 12, 10, 9), (1, 4, 2, 3)); tl.inner_product_tensors(a, b)
a32 = T((64, 12, 10, 9), (1, 2, 3, 4), np.float32); b32 = T((64, 12, 10, 9), (1, 4, 2, 3), np.float32); tl.inner_product_tensors(a32, b32)
torch.cuda.synchronize()
print("ok")
