"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container, where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py small
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py big     # ~20-30 min

It imports ``tensorlib`` from /root/reference/pkg/src (read-only; nothing
is written there) and records what the reference returns:

* ``small.npz``    -- inputs and full outputs of ~250 small seeded cases and
                      the reference tests' known answers, for ttv, ttm,
                      inner, norm, times_vectors and hopm (float64 and int64).
* ``configs.json`` -- for the BASELINE.json configs: sha256 of the
                      reference's output buffers (float64 bytes), sampled
                      values, scalars (norms, inner products) and the full
                      HOPM result of config 4.
* ``cfg1_out.npy`` -- config 1's full 128x64 output.

The GPU box has no /root/reference: tests read only these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import tensorlib as ref  # noqa: E402  (the reference package)

import workloads as W  # noqa: E402


def ref_tensor(buf, shape, layout):
    return ref.DenseTensor.from_memory(tuple(shape), np.asarray(buf).tolist(), layout=tuple(layout))


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


# ------------------------------------------------------------------------------------ small


def draw(rng_np, shape, kind):
    if kind == "int64":
        return rng_np.integers(-9, 10, size=shape).astype(np.int64)
    if kind == "float32":
        return rng_np.uniform(-1.0, 1.0, size=shape).astype(np.float32)
    return rng_np.uniform(-1.0, 1.0, size=shape)


def to_ref_values(buf, kind):
    if kind == "int64":
        return [int(x) for x in np.asarray(buf).reshape(-1)]
    return [float(x) for x in np.asarray(buf, dtype=np.float64).reshape(-1)]


def make_small():
    arrays = {}
    meta = []

    def add(op, **kw):
        i = len(meta)
        entry = {"op": op}
        for k, v in kw.items():
            if isinstance(v, np.ndarray):
                arrays[f"c{i}_{k}"] = v
                entry[k] = f"c{i}_{k}"
            else:
                entry[k] = v
        meta.append(entry)

    rng = random.Random(1234)
    nrng = np.random.default_rng(1234)

    # ttv: random order/extents/layout/mode, float64 + float32 + int64
    for t in range(90):
        kind = "int64" if t % 3 == 2 else ("float32" if t % 6 == 1 else "float64")
        p = rng.randint(2, 5)
        shape = tuple(rng.randint(1, 6) for _ in range(p))
        layout = W.random_layout(p, rng.randint(0, 10**6))
        mode = rng.randint(1, p)
        T = draw(nrng, shape, kind)
        b = draw(nrng, (shape[mode - 1],), kind)
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, layout), kind), layout=layout)
        col = rng.random() < 0.2
        if col:
            B = ref.DenseTensor.from_memory((shape[mode - 1], 1), to_ref_values(b, kind))
        else:
            B = ref.DenseTensor.from_memory((shape[mode - 1],), to_ref_values(b, kind))
        C = ref.ttv(A, B, mode)
        add("ttv", kind=kind, shape=list(shape), layout=list(layout), mode=mode, column=col,
            a=W.layout_buffer(T, layout), b=b, out=np.asarray(C.data, dtype=np.int64 if kind == "int64" else np.float64),
            out_shape=list(C.shape))

    # ttm
    for t in range(60):
        kind = "int64" if t % 3 == 2 else "float64"
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 6) for _ in range(p))
        layout = W.random_layout(p, rng.randint(0, 10**6))
        mode = rng.randint(1, p)
        J = rng.randint(1, 5)
        blayout = (1, 2) if rng.random() < 0.5 else (2, 1)
        T = draw(nrng, shape, kind)
        M = draw(nrng, (J, shape[mode - 1]), kind)
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, layout), kind), layout=layout)
        Bm = ref.DenseTensor.from_memory(M.shape, to_ref_values(W.layout_buffer(M, blayout), kind), layout=blayout)
        C = ref.ttm(A, Bm, mode)
        add("ttm", kind=kind, shape=list(shape), layout=list(layout), mode=mode, blayout=list(blayout),
            a=W.layout_buffer(T, layout), bmat=W.layout_buffer(M, blayout), bshape=list(M.shape),
            out=np.asarray(C.data, dtype=np.int64 if kind == "int64" else np.float64), out_shape=list(C.shape))

    # inner (mixed layouts) and norm
    for t in range(40):
        kind = "int64" if t % 4 == 3 else "float64"
        p = rng.randint(1, 5)
        shape = tuple(rng.randint(1, 6) for _ in range(p))
        la = W.random_layout(p, rng.randint(0, 10**6))
        lb = W.random_layout(p, rng.randint(0, 10**6))
        Ta, Tb = draw(nrng, shape, kind), draw(nrng, shape, kind)
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(Ta, la), kind), layout=la)
        B = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(Tb, lb), kind), layout=lb)
        val = ref.inner_product_tensors(A, B)
        add("inner", kind=kind, shape=list(shape), layout=list(la), blayout=list(lb),
            a=W.layout_buffer(Ta, la), b=W.layout_buffer(Tb, lb), value=val)
    for t in range(20):
        p = rng.randint(1, 5)
        shape = tuple(rng.randint(1, 7) for _ in range(p))
        la = W.random_layout(p, rng.randint(0, 10**6))
        Ta = draw(nrng, shape, "float64")
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(Ta, la), "float64"), layout=la)
        add("norm", kind="float64", shape=list(shape), layout=list(la), a=W.layout_buffer(Ta, la),
            value=ref.frobenius_norm(A))

    # times_vectors: skip form and explicit modes
    for t in range(16):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 5) for _ in range(p))
        la = W.random_layout(p, rng.randint(0, 10**6))
        T = draw(nrng, shape, "float64")
        vs = [draw(nrng, (n,), "float64") for n in shape]
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, la), "float64"), layout=la)
        V = [ref.DenseTensor.from_memory((n,), v.tolist()) for n, v in zip(shape, vs)]
        if t % 2 == 0:
            skip = rng.randint(1, p)
            C = ref.times_vectors(A, V, skip=skip)
            modes = None
        else:
            k = rng.randint(1, p)
            modes = sorted(rng.sample(range(1, p + 1), k))
            C = ref.times_vectors(A, [V[m - 1] for m in modes], modes)
            skip = None
        add("times_vectors", kind="float64", shape=list(shape), layout=list(la), skip=skip, modes=modes,
            a=W.layout_buffer(T, la), vectors=np.concatenate(vs), out=np.asarray(C.data, dtype=np.float64),
            out_shape=list(C.shape))

    # hopm on small random tensors (tol=0 -> exactly max_sweeps sweeps) and default tol
    hopm_cases = [((3, 4, 2), 12, 0.0), ((4, 3), 10, 0.0), ((5, 4, 3, 2), 8, 0.0), ((6, 5, 4), 20, 1e-10),
                  ((3, 3, 3), 1, 1e-10), ((2, 3, 4, 2, 3), 6, 0.0), ((7,), 3, 0.0), ((9, 8, 7), 30, 1e-10)]
    for shape, sweeps, tol in hopm_cases:
        p = len(shape)
        la = W.random_layout(p, rng.randint(0, 10**6))
        T = draw(nrng, shape, "float64")
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, la), "float64"), layout=la)
        st = ref.hopm(A, max_sweeps=sweeps, tol=tol)
        add("hopm", kind="float64", shape=list(shape), layout=list(la), max_sweeps=sweeps, tol=tol,
            a=W.layout_buffer(T, la), u=np.concatenate([np.asarray(u.data, dtype=np.float64) for u in st.u]),
            l=np.asarray(st.l, dtype=np.float64), lambda_history=np.asarray(st.lambda_history, dtype=np.float64),
            sweeps=st.sweeps, converged=st.converged)
    # hopm with custom start vectors
    shape = (4, 5, 3)
    T = draw(nrng, shape, "float64")
    u0 = [draw(nrng, (n,), "float64") for n in shape]
    A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, (1, 2, 3)), "float64"))
    st = ref.hopm(A, max_sweeps=7, tol=0.0, u0=[ref.DenseTensor.from_memory((n,), v.tolist()) for n, v in zip(shape, u0)])
    add("hopm", kind="float64", shape=list(shape), layout=[1, 2, 3], max_sweeps=7, tol=0.0,
        a=W.layout_buffer(T, (1, 2, 3)), u0=np.concatenate(u0),
        u=np.concatenate([np.asarray(u.data, dtype=np.float64) for u in st.u]),
        l=np.asarray(st.l, dtype=np.float64), lambda_history=np.asarray(st.lambda_history, dtype=np.float64),
        sweeps=st.sweeps, converged=st.converged)

    # hopm with track_residuals, and rank_one_compose (hopm.py:114-115, 123-147)
    for shape, sweeps in [((4, 3, 5), 6), ((3, 4), 5), ((2, 3, 4, 2), 4)]:
        p = len(shape)
        la = W.random_layout(p, rng.randint(0, 10**6))
        T = draw(nrng, shape, "float64")
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, la), "float64"), layout=la)
        st = ref.hopm(A, max_sweeps=sweeps, tol=0.0, track_residuals=True)
        B = ref.rank_one_compose(st.scale, st.u)
        add("hopm_resid", kind="float64", shape=list(shape), layout=list(la), max_sweeps=sweeps, tol=0.0,
            a=W.layout_buffer(T, la), residual_history=np.asarray(st.residual_history, dtype=np.float64),
            lambda_history=np.asarray(st.lambda_history, dtype=np.float64),
            u=np.concatenate([np.asarray(u.data, dtype=np.float64) for u in st.u]),
            compose=np.asarray(B.data, dtype=np.float64), residual=ref.residual(A, st))

    # medium cases exercising each kernel regime (contracted stride 1 / strided;
    # small and wide inner blocks; odd extents)
    medium = [((40, 33, 17), (1, 2, 3), 1), ((40, 33, 17), (1, 2, 3), 2), ((40, 33, 17), (3, 2, 1), 1),
              ((40, 33, 17), (2, 3, 1), 3), ((64, 48, 9), (3, 1, 2), 3), ((9, 130, 7, 5), (2, 4, 1, 3), 2),
              ((256, 3, 70), (1, 2, 3), 3), ((5, 300, 11), (2, 1, 3), 2)]
    for shape, layout, mode in medium:
        for kind in ("float64", "float32"):
            T = draw(nrng, shape, kind)
            b = draw(nrng, (shape[mode - 1],), kind)
            A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, layout), kind), layout=layout)
            B = ref.DenseTensor.from_memory((shape[mode - 1],), to_ref_values(b, kind))
            C = ref.ttv(A, B, mode)
            add("ttv", kind=kind, shape=list(shape), layout=list(layout), mode=mode, column=False,
                a=W.layout_buffer(T, layout), b=b, out=np.asarray(C.data, dtype=np.float64), out_shape=list(C.shape))
    medium_ttm = [((24, 20, 18), (1, 2, 3), 2, 13, (1, 2)), ((24, 20, 18), (3, 2, 1), 1, 16, (2, 1)),
                  ((24, 20, 18), (3, 2, 1), 3, 7, (1, 2)), ((3, 33, 5, 17), (1, 2, 3, 4), 2, 16, (1, 2)),
                  ((12, 40, 10), (2, 3, 1), 2, 32, (2, 1))]
    for shape, layout, mode, J, blayout in medium_ttm:
        T = draw(nrng, shape, "float64")
        M = draw(nrng, (J, shape[mode - 1]), "float64")
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, layout), "float64"), layout=layout)
        Bm = ref.DenseTensor.from_memory(M.shape, to_ref_values(W.layout_buffer(M, blayout), "float64"), layout=blayout)
        C = ref.ttm(A, Bm, mode)
        add("ttm", kind="float64", shape=list(shape), layout=list(layout), mode=mode, blayout=list(blayout),
            a=W.layout_buffer(T, layout), bmat=W.layout_buffer(M, blayout), bshape=[J, shape[mode - 1]],
            out=np.asarray(C.data, dtype=np.float64), out_shape=list(C.shape))

    # ttt (contraction.py:337-418): random q, permutations, layouts; transpose; outer product
    for t in range(45):
        kind = "int64" if t % 3 == 2 else ("float32" if t % 3 == 1 else "float64")
        pa, pb = rng.randint(1, 4), rng.randint(1, 4)
        q = rng.randint(0, min(pa, pb))
        phi = tuple(rng.sample(range(1, pa + 1), pa))
        psi = tuple(rng.sample(range(1, pb + 1), pb))
        sa = [rng.randint(1, 5) for _ in range(pa)]
        sb = [rng.randint(1, 5) for _ in range(pb)]
        for k in range(q):
            sb[psi[pb - q + k] - 1] = sa[phi[pa - q + k] - 1]
        la = W.random_layout(pa, rng.randint(0, 10**6))
        lb = W.random_layout(pb, rng.randint(0, 10**6))
        Ta, Tb = draw(nrng, tuple(sa), kind), draw(nrng, tuple(sb), kind)
        A = ref.DenseTensor.from_memory(tuple(sa), to_ref_values(W.layout_buffer(Ta, la), kind), layout=la)
        B = ref.DenseTensor.from_memory(tuple(sb), to_ref_values(W.layout_buffer(Tb, lb), kind), layout=lb)
        C = ref.ttt(A, B, ref.ContractionSpec(q, phi, psi))
        add("ttt", kind=kind, shape=sa, layout=list(la), bshape=sb, blayout=list(lb), q=q, phi=list(phi),
            psi=list(psi), a=W.layout_buffer(Ta, la), b=W.layout_buffer(Tb, lb),
            out=np.asarray(C.data, dtype=np.int64 if kind == "int64" else np.float64), out_shape=list(C.shape))
    for t in range(12):
        kind = "int64" if t % 2 else "float64"
        p = rng.randint(1, 5)
        shape = tuple(rng.randint(1, 5) for _ in range(p))
        la = W.random_layout(p, rng.randint(0, 10**6))
        tau = tuple(rng.sample(range(1, p + 1), p))
        T = draw(nrng, shape, kind)
        A = ref.DenseTensor.from_memory(shape, to_ref_values(W.layout_buffer(T, la), kind), layout=la)
        C = ref.transpose(A, tau)
        add("transpose", kind=kind, shape=list(shape), layout=list(la), tau=list(tau), a=W.layout_buffer(T, la),
            out=np.asarray(C.data, dtype=np.int64 if kind == "int64" else np.float64), out_shape=list(C.shape))
    for sa, sb in [((3,), (4,)), ((2, 3), (4,)), ((2,), (3, 2)), ((1, 3), (2, 1, 2))]:
        Ta, Tb = draw(nrng, sa, "float64"), draw(nrng, sb, "float64")
        A = ref.DenseTensor.from_memory(sa, Ta.reshape(-1, order="F").tolist())
        B = ref.DenseTensor.from_memory(sb, Tb.reshape(-1, order="F").tolist())
        C = ref.outer_product(A, B)
        add("outer", kind="float64", shape=list(sa), bshape=list(sb), a=Ta.reshape(-1, order="F"),
            b=Tb.reshape(-1, order="F"), out=np.asarray(C.data, dtype=np.float64), out_shape=list(C.shape))

    # known answers restated from the reference's own tests
    I2 = ref.DenseTensor((2, 2))
    I2[0, 0] = 1
    I2[1, 1] = 1
    kat = {
        # test_contraction.py:78-80
        "ttv_identity_row_sums": ref.ttv(I2, ref.DenseTensor((2,), fill_value=1), 2).data,
        # test_contraction.py:82-86
        "ttv_counting": ref.ttv(ref.DenseTensor((2, 3, 2), fill_value=1), ref.DenseTensor((3,), fill_value=1), 2).data,
        # test_contraction.py:295-296
        "norm_all_ones_222": ref.frobenius_norm(ref.DenseTensor((2, 2, 2), fill_value=1)),
        # test_contraction.py:326-330
        "times_vectors_full_ones": ref.times_vectors(ref.DenseTensor((2, 3, 2), fill_value=1),
                                                     [ref.DenseTensor((n,), fill_value=1) for n in (2, 3, 2)],
                                                     [1, 2, 3]).data,
    }
    st = ref.hopm(ref.DenseTensor.from_memory((3,), [3.0, 0.0, 4.0]))  # test_hopm.py:46-50
    kat["hopm_order_one"] = {"l": st.l, "u": st.u[0].data}
    try:
        ref.hopm(ref.DenseTensor((2, 3)))  # test_hopm.py:52-55
    except ref.DegenerateInputError as e:
        kat["hopm_zero_degenerate"] = [e.sweep, e.mode]

    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump({"cases": meta, "kat": kat, "generator": "tests/golden/make_golden.py small",
                   "reference": "/root/reference/pkg/src/tensorlib 0.1.0"}, f, indent=1)
    print(f"small: {len(meta)} cases")


# -------------------------------------------------------------------------------------- big


def make_big(which):
    path = os.path.join(HERE, "configs.json")
    out = json.load(open(path)) if os.path.exists(path) else {}

    def save():
        with open(path, "w") as f:
            json.dump(out, f, indent=1)

    def sample(arr, n=64):
        idx = np.random.default_rng(99).integers(0, arr.size, size=n)
        return {"idx": idx.tolist(), "val": [float(arr[i]) for i in idx]}

    if "cfg1" in which:
        T, b = W.cfg1()
        t0 = time.time()
        A = ref_tensor(W.layout_buffer(T, (1, 2, 3)), T.shape, (1, 2, 3))
        C = ref.ttv(A, ref.DenseTensor.from_memory((96,), b.tolist()), 2)
        dt = time.time() - t0
        c = np.asarray(C.data, dtype=np.float64)
        np.save(os.path.join(HERE, "cfg1_out.npy"), c)
        out["cfg1"] = {"sha256": sha(c), "shape": list(C.shape), "input_sha256": sha(T), "ref_seconds": dt}
        save()
        print("cfg1 done", dt)

    if "cfg5" in which:
        for seed in (0, 5):
            T, v, M, layout = W.cfg5(seed)
            A = ref_tensor(W.layout_buffer(T, layout), T.shape, layout)
            t0 = time.time()
            C1 = ref.ttv(A, ref.DenseTensor.from_memory((9,), v.tolist()), 5)
            t1 = time.time()
            Bm = ref.DenseTensor.from_memory(M.shape, W.layout_buffer(M, (1, 2)).tolist())
            C2 = ref.ttm(C1, Bm, 2)
            t2 = time.time()
            nrm = ref.frobenius_norm(C2)
            t3 = time.time()
            c1 = np.asarray(C1.data, dtype=np.float64)
            c2 = np.asarray(C2.data, dtype=np.float64)
            out[f"cfg5_seed{seed}"] = {
                "layout": list(layout), "input_sha256": sha(T),
                "ttv_sha256": sha(c1), "ttv_sample": sample(c1), "ttv_shape": list(C1.shape),
                "ttm_sha256": sha(c2), "ttm_sample": sample(c2), "ttm_shape": list(C2.shape),
                "norm": nrm, "ref_seconds": {"ttv": t1 - t0, "ttm": t2 - t1, "norm": t3 - t2},
            }
            del A, C1, C2, c1, c2
            save()
            print("cfg5", seed, "done", t3 - t0)

    if "cfg2" in which:
        T, vecs, T2 = W.cfg2()
        res = out.get("cfg2", {})
        for name, layout in W.CFG2_LAYOUTS.items():
            buf = W.layout_buffer(T, layout)
            A = ref_tensor(buf, T.shape, layout)
            del buf
            for mode in (1, 2, 3, 4):
                t0 = time.time()
                C = ref.ttv(A, ref.DenseTensor.from_memory((128,), [float(x) for x in vecs[mode - 1]]), mode)
                dt = time.time() - t0
                c = np.asarray(C.data, dtype=np.float64)
                res[f"ttv_{name}_q{mode}"] = {"sha256": sha(c), "sample": sample(c), "ref_seconds": dt,
                                              "f32_sha256": sha(c.astype(np.float32))}
                print("cfg2", name, mode, dt, flush=True)
            if name == "first":
                t0 = time.time()
                res["norm_first"] = {"value": ref.frobenius_norm(A), "ref_seconds": time.time() - t0}
                buf2 = W.layout_buffer(T2, layout)
                B = ref_tensor(buf2, T2.shape, layout)
                del buf2
                t0 = time.time()
                res["inner_first_first"] = {"value": ref.inner_product_tensors(A, B), "ref_seconds": time.time() - t0}
                del B
                last = W.CFG2_LAYOUTS["last"]
                buf2 = W.layout_buffer(T2, last)
                B = ref_tensor(buf2, T2.shape, last)
                del buf2
                t0 = time.time()
                res["inner_first_last"] = {"value": ref.inner_product_tensors(A, B), "ref_seconds": time.time() - t0}
                del B
            out["cfg2"] = res
            save()
            del A

    if "cfg4" in which:
        T, vs = W.cfg4()
        A = ref_tensor(W.layout_buffer(T, (1, 2, 3)), T.shape, (1, 2, 3))
        t0 = time.time()
        st = ref.hopm(A, max_sweeps=50, tol=0.0)
        dt = time.time() - t0
        out["cfg4"] = {"lambda_history": st.lambda_history, "l": st.l, "sweeps": st.sweeps,
                       "converged": st.converged, "u": [u.data for u in st.u], "ref_seconds": dt,
                       "input_sha256": sha(T)}
        save()
        print("cfg4 done", dt)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        make_small()
    else:
        make_big(sys.argv[2:] or ["cfg1", "cfg5", "cfg2", "cfg4"])
