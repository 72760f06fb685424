"""Quick per-op timing on the GPU box (development aid; bench.py is the contract)."""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch

import paper_1711_10912_b200 as tl
import workloads as W

HBM = 6456.2


def timeit(fn, iters=10, warm=3, reps=8):
    """Device time per call: `reps` calls in one CUDA graph (no host overhead)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    del g
    return float(np.median(ts)), float(np.min(ts))


def timeit_eager(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(np.min(ts))


def main(which):
    if "cfg2" in which:
        T, vecs, T2 = W.cfg2()
        vs = [tl.DenseTensor.from_memory((128,), v) for v in vecs]
        for name, layout in W.CFG2_LAYOUTS.items():
            A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, layout), layout=layout)
            for mode in (1, 2, 3, 4):
                med, mn = timeit(lambda: tl.ttv(A, vs[mode - 1], mode))
                byts = 4 * (2**28 + 128 + 2**21)
                print(f"cfg2 ttv {name:5s} q={mode}: {med*1e3:8.1f} us  {byts/med/1e6:7.1f} GB/s  ({byts/med/1e6/HBM:.2f} of HBM)", flush=True)
            if name == "first":
                med, _ = timeit(lambda: tl.frobenius_norm_device(A) if hasattr(tl, "frobenius_norm_device") else tl.contraction.frobenius_norm_device(A))
                print(f"cfg2 norm: {med*1e3:8.1f} us {4*2**28/med/1e6:7.1f} GB/s", flush=True)
                B = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T2, layout), layout=layout, dtype="float32")
                med, _ = timeit(lambda: tl.contraction.inner_product_device(A, B))
                print(f"cfg2 inner ff: {med*1e3:8.1f} us {8*2**28/med/1e6:7.1f} GB/s", flush=True)
                Bl = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T2, (4, 3, 2, 1)), layout=(4, 3, 2, 1))
                med, _ = timeit(lambda: tl.contraction.inner_product_device(A, Bl))
                print(f"cfg2 inner fl: {med*1e3:8.1f} us {8*2**28/med/1e6:7.1f} GB/s", flush=True)
                del B, Bl
                from paper_1711_10912_b200.tensor import _copy
                import paper_1711_10912_b200._abi as abi

                for lay in ((4, 3, 2, 1), (3, 1, 2, 4)):
                    out = torch.empty_like(A.buffer)
                    cd = abi.make_desc(A.shape, tl.compute_strides(A.shape, lay), abi.TL_F32)
                    med, _ = timeit(lambda: _copy(A.desc(), A.buffer, cd, out))
                    print(f"cfg2 relayout first->{lay}: {med*1e3:8.1f} us {8*2**28/med/1e6:7.1f} GB/s", flush=True)
                    del out
            del A
            torch.cuda.empty_cache()
    if "cfg5" in which:
        for seed in (0, 5):
            T, v, M, layout = W.cfg5(seed)
            A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, layout), layout=layout)
            V = tl.DenseTensor.from_memory((9,), v)
            Bm = tl.DenseTensor.from_memory(M.shape, W.layout_buffer(M, (1, 2)))
            med, _ = timeit(lambda: tl.ttv(A, V, 5))
            byts = 8 * (96940800 + 9 + 96940800 // 9)
            print(f"cfg5 seed{seed} ttv: {med*1e3:8.1f} us {byts/med/1e6:7.1f} GB/s", flush=True)
            C1 = tl.ttv(A, V, 5)
            med, _ = timeit(lambda: tl.ttm(C1, Bm, 2))
            byts = 8 * (10771200 + 528 + 5222400)
            print(f"cfg5 seed{seed} ttm: {med*1e3:8.1f} us {byts/med/1e6:7.1f} GB/s", flush=True)
            C2 = tl.ttm(C1, Bm, 2)
            med, _ = timeit(lambda: tl.contraction.frobenius_norm_device(C2))
            print(f"cfg5 seed{seed} norm: {med*1e3:8.1f} us {8*5222400/med/1e6:7.1f} GB/s", flush=True)
            del A, C1, C2
            torch.cuda.empty_cache()
    if "cfg4" in which:
        T, _ = W.cfg4()
        A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3)))
        r = tl.HopmRunner(A, max_sweeps=50, tol=0.0)
        med, mn = timeit_eager(r.launch, iters=5, warm=2)
        print(f"cfg4 hopm 50 sweeps: {med:.3f} ms -> {50/med*1e3:.0f} sweeps/s; 2-pass bytes frac "
              f"{2*8*64e6*50/(med*1e-3)/1e9/HBM:.2f}", flush=True)
        st = r.state()
        print("  lambda50", st.lambda_history[-1])
        r.close()
    if "cfg3" in which:
        A_, B_ = W.cfg3()
        for layout in ((1, 2, 3), (3, 2, 1)):
            A = tl.DenseTensor.from_memory(A_.shape, W.layout_buffer(A_, layout), layout=layout)
            Bm = tl.DenseTensor.from_memory(B_.shape, W.layout_buffer(B_, (1, 2)))
            for mode in (1, 2, 3):
                med, _ = timeit_eager(lambda: tl.ttm(A, Bm, mode), iters=3, warm=1)
                fl = 2 * 512**3 * 384
                print(f"cfg3 ttm {layout} q={mode}: {med:.3f} ms {fl/med/1e9:.2f} TFLOP/s", flush=True)
            del A
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg5", "cfg4", "cfg3"])
