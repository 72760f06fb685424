"""bench.py -- the driver's benchmark contract for the tensorlib B200 hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], the config the headline metric is
quoted on): the ttv sweep over modes 1..4 of an order-4 float32 128^4
tensor (1 GiB) in first-order, last-order and seeded-permutation layouts,
plus the inner product of two such tensors and the Frobenius norm.  One
step = those 14 operations.  value = algorithmic HBM bytes of the step
(each operand read once, each output written once) divided
by the device time of the step, in GB/s.  Inputs are 1 GiB each (8x the
126 MB L2), so no L2 flush is needed between iterations.

Multi-GPU: one process per GPU (torchrun); every rank runs its own copy of
the workload (independent units, no data-path collective) -> weak scaling;
the step time is the max over ranks (NCCL all-reduce of the event time).

Also measured on rank 0 (``components``): config 1 ttv, config 3 ttm
(FP64 DMMA TFLOP/s, 6 cases), config 4 HOPM (sweeps/s, 50-sweep graph),
config 5 ttv -> ttm -> norm chain.

``--impl reference`` times the reference's CPU algorithm (the pinned C
oracle port, oracle/tl_oracle.c, all host threads) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "ttv/norm HBM GB/s, ttm FP64 TFLOP/s (fraction of B200 roofline); HOPM iters/s"
N4 = 128 ** 4
TTV_BYTES = 4 * (N4 + 128 + N4 // 128)       # per ttv launch
NORM_BYTES = 4 * N4
INNER_BYTES = 8 * N4
STEP_BYTES = 12 * TTV_BYTES + NORM_BYTES + INNER_BYTES
FP64_PEAK_TFLOPS = 37.0  # DMMA/DFMA, measured by tools/fp64_probe.cu (profiles/fp64_probe_r01.txt)
L2_FLUSH_BYTES = 512 << 20  # > 4x the 126 MB L2: written between cold-timed launches


def cfg2_config(world):
    """The workload's config object -- identical for both arms."""
    return {"workload": "cfg2: ttv q=1..4 x {first,last,perm(3,1,2,4)} + inner + norm, f32 128^4 (1 GiB)",
            "step_bytes": STEP_BYTES, "l2": "inputs 1 GiB each > 126 MB L2 (no flush needed)",
            "parallelism": f"{world} independent replicas (weak scaling, no collective)"}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def hbm_peak():
    p = measured_peaks().get("hbm_gbs")
    return (float(p), "measured") if p else (6650.0, "fallback")


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sms:
            return None
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sms)}


# ----------------------------------------------------------------- distributed
def dist_setup(n_gpus, backend="nccl"):
    """One process per GPU (torchrun env); returns (world, rank, local_rank)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def dist_max(x, world):
    """Max over ranks (the step time of a weak-scaled run is the slowest rank's)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(step_bytes, world, ms_max):
    """Whole-job throughput of `world` independent replicas, GB/s."""
    return world * step_bytes / (ms_max * 1e-3) / 1e9


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ---------------------------------------------------------------- b200 workload
class Cfg2Workload:
    """Device-resident inputs for one step (3 layouts of T, T2, vectors)."""

    def __init__(self):
        import paper_1711_10912_b200 as tl

        self.tl = tl
        T, vecs, T2 = W.cfg2()
        self.host = {}
        self.A = {}
        for name, layout in W.CFG2_LAYOUTS.items():
            buf = W.layout_buffer(T, layout)
            self.host[name] = (buf, layout)
            self.A[name] = tl.DenseTensor.from_memory(T.shape, buf, layout=layout)
        self.host_T2 = W.layout_buffer(T2, (1, 2, 3, 4))
        self.B = tl.DenseTensor.from_memory(T.shape, self.host_T2, layout=(1, 2, 3, 4))
        self.vecs = [tl.DenseTensor.from_memory((128,), v) for v in vecs]
        self.host_vecs = vecs
        del T, T2

    def step(self, ev_ttv=None):
        """12 ttv + norm + inner; results stay on the device."""
        tl = self.tl
        import paper_1711_10912_b200.contraction as C

        outs = []
        for name in W.CFG2_LAYOUTS:
            A = self.A[name]
            for mode in (1, 2, 3, 4):
                if ev_ttv is not None:
                    ev_ttv.begin()
                outs.append(tl.ttv(A, self.vecs[mode - 1], mode))
                if ev_ttv is not None:
                    ev_ttv.end()
        nrm = C.frobenius_norm_device(self.A["first"])
        ip = C.inner_product_device(self.A["first"], self.B)
        return outs, nrm, ip


class EventPairs:
    """CUDA events around each launch of one kernel family on its stream."""

    def __init__(self):
        import torch

        self.torch = torch
        self.pairs = []
        self.cur = None

    def begin(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self.cur = e

    def end(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self.pairs.append((self.cur, e))

    def mean_ms(self):
        return statistics.mean(a.elapsed_time(b) for a, b in self.pairs)


def time_device(fn, steps, warmup, world=1):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        fn()
    t1.record()
    torch.cuda.synchronize()
    barrier(world)
    return t0.elapsed_time(t1) / steps


def e2e_step(wl, relayout_on_device=False):
    """Public API end to end, every step from pinned host memory.

    Default (the reference arm's input contract, three host buffers per
    step): the first-order, last-order and permuted buffers of T and the
    first-order T2 are uploaded (copy stream; each layout's four ttvs start
    as soon as its buffer has landed), the 14 ops run, and every ttv
    output plus both scalars are read back to the host (a third stream, so
    downloads overlap uploads on the other copy engine).

    ``relayout_on_device``: only T and T2 are uploaded; the last-order and
    permuted copies are made on the device with DenseTensor.relayout."""
    import torch

    tl = wl.tl
    h2d = d2h = 0
    cur = torch.cuda.current_stream()
    up, down = wl.up_stream, wl.down_stream
    up.wait_stream(cur)
    vecs = [tl.DenseTensor.from_memory((128,), v) for v in wl.pinned_vecs]
    h2d += 4 * 128 * 4
    A, ready = {}, {}
    names = ["first"] if relayout_on_device else list(W.CFG2_LAYOUTS)
    with torch.cuda.stream(up):
        for name in names:
            buf, layout = wl.pinned[name]
            A[name] = tl.DenseTensor.from_memory(W.CFG2_SHAPE, buf, layout=layout)
            h2d += buf.numel() * 4
            ready[name] = torch.cuda.Event()
            ready[name].record(up)
        B = tl.DenseTensor.from_memory(W.CFG2_SHAPE, wl.pinned_T2, layout=(1, 2, 3, 4))
        h2d += wl.pinned_T2.numel() * 4
        ready["T2"] = torch.cuda.Event()
        ready["T2"].record(up)
    for t in list(A.values()) + [B]:
        t.buffer.record_stream(cur)
    cur.wait_event(ready["first"])
    if relayout_on_device:
        for name, layout in W.CFG2_LAYOUTS.items():
            if name != "first":
                t = A["first"].copy()
                t.relayout(layout)
                A[name] = t
    res = []
    for name in W.CFG2_LAYOUTS:
        if name in ready:
            cur.wait_event(ready[name])
        for mode in (1, 2, 3, 4):
            c = tl.ttv(A[name], vecs[mode - 1], mode)
            done = torch.cuda.Event()
            done.record(cur)
            down.wait_event(done)
            with torch.cuda.stream(down):
                host = torch.empty(c.size, dtype=c.dtype, pin_memory=True)
                host.copy_(c.buffer, non_blocking=True)
            c.buffer.record_stream(down)
            res.append(host)
            d2h += c.size * 4
    nrm = C_norm(A["first"])
    cur.wait_event(ready["T2"])
    ip = C_inner(A["first"], B)
    scal = torch.empty(2, dtype=torch.float64, pin_memory=True)
    scal[0:1].copy_(nrm, non_blocking=True)
    scal[1:2].copy_(ip, non_blocking=True)
    d2h += 16
    torch.cuda.synchronize()
    return h2d, d2h, (res, scal)


def C_norm(a):
    import paper_1711_10912_b200.contraction as C

    return C.frobenius_norm_device(a)


def C_inner(a, b):
    import paper_1711_10912_b200.contraction as C

    return C.inner_product_device(a, b)


def time_e2e(wl, steps, warmup, world, relayout_on_device=False):
    import torch

    for _ in range(warmup):  # also warms the pinned host-buffer cache
        e2e_step(wl, relayout_on_device)
    barrier(world)
    torch.cuda.synchronize()
    te = time.perf_counter()
    n = max(1, min(5, steps))
    for _ in range(n):
        h2d, d2h, res = e2e_step(wl, relayout_on_device)
        del res
    dt = dist_max((time.perf_counter() - te) / n, world)
    return {"value": round(world * STEP_BYTES / dt / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(dt * 1e3, 2)}


# ------------------------------------------------------------------ components
def components(args, wl=None):
    """Per-config numbers on rank 0 (each a median of CUDA-event timings)."""
    import torch

    import paper_1711_10912_b200 as tl
    import paper_1711_10912_b200.contraction as C

    out = {}

    def med(fn, iters=5, warm=2, reps=10):
        """Median device time of one call: `reps` calls captured in a CUDA
        graph and replayed, so host launch overhead does not count."""
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
        g.replay()
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
        return statistics.median(ts)

    flush_buf = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    flush_sink = torch.empty(1, dtype=torch.float32, device="cuda")

    def flush_l2(r):
        """Evict L2 by READING 512 MB (4x L2): clean lines, so the timed op
        pays no write-back of the flush's own data (a write flush would leave
        ~126 MB of dirty lines for the op to evict)."""
        torch.sum(flush_buf, dim=0, keepdim=True, out=flush_sink)

    def cold(fn, reps=20, iters=5):
        """Device time of one launch with a cold L2: a CUDA graph of `reps`
        x [512 MB read (4x L2), fn] minus a graph of `reps` x [the same
        read], divided by `reps` -- no event or host launch overhead in the
        number (an event pair around a single eager launch adds ~6 us on
        this box: tools/experiments/red_probe.cu)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
            fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graphs = []
        for with_fn in (True, False):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for r in range(reps):
                    flush_l2(r)
                    if with_fn:
                        fn()
            graphs.append(g)
        ts = {True: [], False: []}
        for _ in range(iters):
            for with_fn, g in zip((True, False), graphs):
                g.replay()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                ts[with_fn].append(a.elapsed_time(b))
        del graphs
        return (statistics.median(ts[True]) - statistics.median(ts[False])) / reps

    def med_eager(fn, iters=5, warm=2):
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
        return statistics.median(ts)

    peak, _ = hbm_peak()
    # config 2 extras: the first x last mixed-layout inner product (SURVEY
    # a6) and the layout conversions the e2e relies on (relayout/transpose)
    if wl is not None:
        Af, Al = wl.A["first"], wl.A["last"]
        ms = med(lambda: C.inner_product_device(Af, Al), iters=5, reps=5)
        out["cfg2_inner_first_x_last_us"] = round(ms * 1e3, 1)
        out["cfg2_inner_first_x_last_frac_hbm"] = round(INNER_BYTES / (ms * 1e-3) / 1e9 / peak, 3)
        relay = {}
        for name, tau in (("first_to_last", (4, 3, 2, 1)), ("first_to_perm3124", (3, 1, 2, 4)),
                          ("first_to_2134", (2, 1, 3, 4))):
            ms = med(lambda: tl.transpose(Af, tau), iters=5, reps=5)
            relay[name] = {"us": round(ms * 1e3, 1), "frac_hbm": round(2 * 4 * N4 / (ms * 1e-3) / 1e9 / peak, 3)}
        out["cfg2_transpose"] = relay
        torch.cuda.empty_cache()
    # config 1
    T, b = W.cfg1()
    A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3)))
    V = tl.DenseTensor.from_memory((96,), b)
    ms = med(lambda: tl.ttv(A, V, 2), iters=20)
    out["cfg1_ttv_us"] = round(ms * 1e3, 2)
    # config 3: ttm FP64
    A_, B_ = W.cfg3()
    Bm = tl.DenseTensor.from_memory(B_.shape, W.layout_buffer(B_, (1, 2)))
    tf = {}
    for lname, layout in (("first", (1, 2, 3)), ("last", (3, 2, 1))):
        A = tl.DenseTensor.from_memory(A_.shape, W.layout_buffer(A_, layout), layout=layout)
        for mode in (1, 2, 3):
            ms = med_eager(lambda: tl.ttm(A, Bm, mode), iters=3, warm=1)
            tf[f"{lname}_q{mode}"] = round(2 * 512 ** 3 * 384 / (ms * 1e-3) / 1e12, 2)
        del A
        torch.cuda.empty_cache()
    out["cfg3_ttm_tflops"] = tf
    out["cfg3_ttm_tflops_min"] = min(tf.values())
    out["cfg3_ttm_frac_fp64_peak_min"] = round(min(tf.values()) / FP64_PEAK_TFLOPS, 3)
    # the same contraction as a general ttt (reduce_ttm_to_ttt: A's mode 2 with
    # B's columns): two device relayouts + the GETT (contraction.py:337-369)
    A1 = tl.DenseTensor.from_memory(A_.shape, W.layout_buffer(A_, (1, 2, 3)))
    spec = tl.reduce_ttm_to_ttt(3, 2)
    ms = med_eager(lambda: tl.ttt(A1, Bm, spec), iters=3, warm=1)
    out["cfg3_ttt_q2_ms"] = round(ms, 3)
    out["cfg3_ttt_q2_tflops"] = round(2 * 512 ** 3 * 384 / (ms * 1e-3) / 1e12, 2)
    del A1
    torch.cuda.empty_cache()
    # the same shape in float32 storage (widened onto the FP64 tensor cores;
    # an extension: the reference has no float32)
    A32 = tl.DenseTensor.from_memory(A_.shape, W.layout_buffer(A_, (1, 2, 3)).astype(np.float32))
    B32 = Bm.to(torch.float32)
    ms = med_eager(lambda: tl.ttm(A32, B32, 2), iters=3, warm=1)
    out["cfg3_f32_first_q2_tflops"] = round(2 * 512 ** 3 * 384 / (ms * 1e-3) / 1e12, 2)
    del A32, B32, A_
    # config 4: HOPM
    T, _ = W.cfg4()
    A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3)))
    del T
    r = tl.HopmRunner(A, max_sweeps=50, tol=0.0)
    ms = med_eager(r.launch, iters=5, warm=2)
    st = r.state()
    r.close()
    sps = 50 / (ms * 1e-3)
    out["cfg4_hopm_sweeps_per_s"] = round(sps, 1)
    out["cfg4_hopm_lambda50"] = st.lambda_history[-1]
    out["cfg4_hopm_frac_hbm_2pass"] = round(sps * 2 * 8 * 400 ** 3 / 1e9 / peak, 3)
    del A
    torch.cuda.empty_cache()
    # config 5 chain (both seeded layouts)
    for seed in (0, 5):
        T, v, M, layout = W.cfg5(seed)
        A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, layout), layout=layout)
        del T
        Vv = tl.DenseTensor.from_memory((9,), v)
        Bm5 = tl.DenseTensor.from_memory(M.shape, W.layout_buffer(M, (1, 2)))
        t_ttv = med(lambda: tl.ttv(A, Vv, 5))
        C1 = tl.ttv(A, Vv, 5)
        os.environ["TL_FUSED_NORM"] = "0"  # the ttm alone (no fused norm epilogue)
        t_ttm = cold(lambda: tl.ttm(C1, Bm5, 2))
        t_ttm_warm = med(lambda: tl.ttm(C1, Bm5, 2))
        os.environ.pop("TL_FUSED_NORM")
        C2 = tl.ttm(C1, Bm5, 2).copy()  # a copy: the standalone norm kernel, not ttm's fused value
        t_nrm = cold(lambda: C.frobenius_norm_device(C2))
        t_nrm_warm = med(lambda: C.frobenius_norm_device(C2))

        def chain():
            c1 = tl.ttv(A, Vv, 5)
            return C.frobenius_norm_device(tl.ttm(c1, Bm5, 2))

        # the whole config as the reference states it: ttv -> ttm -> norm of
        # the result, from a cold L2 (the intermediates then stay L2-resident
        # where they fit, as in any run)
        t_chain = cold(chain)  # the norm comes from ttm's fused epilogue
        os.environ["TL_FUSED_NORM"] = "0"
        t_chain_unfused = cold(chain)  # ttm, then the norm kernel over its output
        os.environ.pop("TL_FUSED_NORM")
        n5 = 96940800
        chain_bytes = 8 * (n5 + 9 + n5 // 9) + 8 * (10771200 + 528 + 5222400) + 8 * 5222400
        out[f"cfg5_seed{seed}"] = {
            "layout": list(layout),
            "ttv_us": round(t_ttv * 1e3, 1), "ttv_frac_hbm": round(8 * (n5 + 9 + n5 // 9) / (t_ttv * 1e-3) / 1e9 / peak, 3),
            "ttm_us_cold": round(t_ttm * 1e3, 1),
            "ttm_frac_hbm_cold": round(8 * (10771200 + 528 + 5222400) / (t_ttm * 1e-3) / 1e9 / peak, 3),
            "ttm_us_l2warm": round(t_ttm_warm * 1e3, 1),
            "norm_us_cold": round(t_nrm * 1e3, 1),
            "norm_frac_hbm_cold": round(8 * 5222400 / (t_nrm * 1e-3) / 1e9 / peak, 3),
            "norm_us_l2warm": round(t_nrm_warm * 1e3, 1),
            "chain_us_cold": round(t_chain * 1e3, 1),
            "chain_us_cold_norm_kernel": round(t_chain_unfused * 1e3, 1),
            "chain_frac_hbm": round(chain_bytes / (t_chain * 1e-3) / 1e9 / peak, 3),
        }
        del A, C1, C2
        torch.cuda.empty_cache()
    # north_star "across all layouts and modes": the config-5 ttm operand shape
    # (3,33,5,17,2,640) x a 16-row matrix in the first-order and three seeded
    # permutation layouts, every mode (24 ttms; the full tables over all configs
    # are tools/experiments/config_sweep.py -> profiles/config_sweep_*.md)
    from paper_1711_10912_b200.layout import TensorMeta
    shape5 = (3, 33, 5, 17, 2, 640)
    n5m = int(np.prod(shape5))
    g = torch.Generator(device="cuda").manual_seed(11)
    A0 = tl.DenseTensor._wrap(TensorMeta(shape5), torch.rand(n5m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
    Ms = [tl.DenseTensor._wrap(TensorMeta((16, k)), torch.randn(16 * k, dtype=torch.float64, device="cuda", generator=g))
          for k in shape5]
    refs = [tl.ttm(A0, Ms[m], m + 1).buffer.clone() for m in range(6)]
    fr, same = [], True
    for lay in [tuple(range(1, 7))] + [W.random_layout(6, sd) for sd in (0, 1, 2)]:
        Ap = tl.DenseTensor._wrap(TensorMeta(shape5), A0.buffer.clone())
        Ap.relayout(lay)
        for m in range(6):
            same = same and bool(torch.equal(tl.ttm(Ap, Ms[m], m + 1).buffer, refs[m]))
            t = med(lambda: tl.ttm(Ap, Ms[m], m + 1), iters=3, warm=1, reps=5)
            nb = 8 * (n5m + 16 * shape5[m] + n5m // shape5[m] * 16)
            fr.append(nb / (t * 1e-3) / 1e9 / peak)
        del Ap
    fr.sort()
    out["cfg5_ttm_every_layout_mode"] = {"cases": len(fr), "frac_hbm_min": round(fr[0], 3),
                                         "frac_hbm_median": round(fr[len(fr) // 2], 3), "frac_hbm_max": round(fr[-1], 3),
                                         "bit_identical_across_layouts": same}
    del A0, Ms, refs
    torch.cuda.empty_cache()
    return out


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture summary (profiles/), if present."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        s = json.load(open(path))
        return s.get("ttv_dram_bytes_per_launch")
    except Exception:
        return None


# --------------------------------------------------------------------- CPU arms
def cpu_sweep(T_bufs, T2buf, vecs, nthreads):
    """The reference algorithm (oracle port) over the cfg2 step on the host."""
    from oracle import oracle as O

    for name, (buf, layout) in T_bufs.items():
        st = W.compute_strides(W.CFG2_SHAPE, layout)
        for mode in (1, 2, 3, 4):
            O.ttv(buf, W.CFG2_SHAPE, st, vecs[mode - 1], mode, nthreads=nthreads)
    first = T_bufs["first"][0]
    O.inner_flat_mt(first, first, nthreads)
    O.inner_flat_mt(first, T2buf, nthreads)


def cpu_inputs():
    T, vecs, T2 = W.cfg2()
    bufs = {name: (W.layout_buffer(T, layout), layout) for name, layout in W.CFG2_LAYOUTS.items()}
    return bufs, W.layout_buffer(T2, (1, 2, 3, 4)), vecs


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle import oracle as O

    nthreads = O.max_threads()
    bufs, T2buf, vecs = cpu_inputs()
    for _ in range(args.warmup):
        cpu_sweep(bufs, T2buf, vecs, nthreads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_sweep(bufs, T2buf, vecs, nthreads)
    dt = (time.perf_counter() - t0) / args.steps
    value = STEP_BYTES / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 storage, f64 arithmetic", "data": "synthetic (seeded)",
        "config": cfg2_config(world),
        "cpu_baseline": {"value": round(value, 2), "unit": "GB/s", "cores": nthreads, "kind": "port",
                         "sample": "full cfg2 step per timed step (oracle/tl_oracle.c, OpenMP over outputs)"},
        "e2e": {"value": round(value, 2), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample():
    """Bounded CPU sample on rank 0: one ttv per layout (modes 1, 2, 3) +
    norm with the oracle port on all host threads, scaled to GB/s."""
    from oracle import oracle as O

    nthreads = O.max_threads()
    bufs, T2buf, vecs = cpu_inputs()
    t0 = time.perf_counter()
    done = 0
    for (name, (buf, layout)), mode in zip(bufs.items(), (1, 2, 3)):
        O.ttv(buf, W.CFG2_SHAPE, W.compute_strides(W.CFG2_SHAPE, layout), vecs[mode - 1], mode, nthreads=nthreads)
        done += TTV_BYTES
    O.inner_flat_mt(bufs["first"][0], bufs["first"][0], nthreads)
    done += NORM_BYTES
    dt = time.perf_counter() - t0
    return {"value": round(done / dt / 1e9, 2), "unit": "GB/s", "cores": nthreads, "kind": "port",
            "sample": "3 of the 12 cfg2 ttvs (first q1, last q2, perm q3) + norm, oracle/tl_oracle.c"}


# -------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-components", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch

    torch.cuda.set_device(local)
    wl = Cfg2Workload()
    torch.cuda.synchronize()

    # timed region: K device-resident steps, events around each ttv launch
    ev = EventPairs()
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        wl.step(ev_ttv=ev)
    t1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier(world)
    ms_local = t0.elapsed_time(t1) / args.steps
    ms = dist_max(ms_local, world)
    ttv_ms = ev.mean_ms()
    value = replica_value(STEP_BYTES, world, ms)

    # end to end through the public API (pinned host buffers, copies inside)
    e2e = e2e_relayout = None
    if not args.no_e2e:
        wl.pinned = {name: (torch.from_numpy(buf).pin_memory(), layout) for name, (buf, layout) in wl.host.items()}
        wl.pinned_T2 = torch.from_numpy(wl.host_T2).pin_memory()
        wl.pinned_vecs = [torch.from_numpy(v).pin_memory() for v in wl.host_vecs]
        wl.up_stream, wl.down_stream = torch.cuda.Stream(), torch.cuda.Stream()
        e2e = time_e2e(wl, args.steps, args.warmup, world)
        e2e_relayout = time_e2e(wl, args.steps, args.warmup, world, relayout_on_device=True)
        e2e_relayout["note"] = "T and T2 uploaded; last-order and permuted copies made on the device (relayout)"
        e2e["note"] = "the reference arm's inputs: three host layout buffers of T + T2 uploaded every step"

    if rank != 0:
        barrier(world)
        return
    peak, peak_src = hbm_peak()
    achieved = TTV_BYTES / (ttv_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 storage, f64 arithmetic (bit-exact ttv folds)",
        "data": "synthetic (seeded numpy PCG64; tests/workloads.py)",
        "config": cfg2_config(world),
        "roofline": {"bound": "hbm", "kernel": "ttv (12 launches/step, mean)", "achieved": round(achieved, 1),
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "algorithmic_bytes_per_launch": TTV_BYTES, "mean_launch_us": round(ttv_ms * 1e3, 2),
                     "traffic": ncu_traffic()},
        "gpu_launches": 14 * args.steps,
        "clocks": clk,
        "e2e": e2e,
        "e2e_device_relayout": e2e_relayout,
    }
    if not args.no_components:
        try:
            line["components"] = components(args, wl)
        except Exception as exc:  # keep the headline line even if a component fails
            line["components"] = {"error": repr(exc)}
    if not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline_sample()
        except Exception as exc:
            line["cpu_baseline"] = {"error": repr(exc)}
    print(json.dumps(line), flush=True)
    barrier(world)


if __name__ == "__main__":
    main()
