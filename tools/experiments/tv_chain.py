"""times_vectors: one cooperative launch (chain) vs one ttv launch per vector.
Device time per call (CUDA graph of 10 calls, median of 5 replays)."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path[:0] = [".", "tests"]
import paper_1711_10912_b200 as tl  # noqa: E402
import workloads as W  # noqa: E402


def med(fn, reps=10, iters=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    return statistics.median(ts)


res = {}
T, vecs, _ = W.cfg2()
A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3, 4)))
del T
V = [tl.DenseTensor.from_memory((128,), v) for v in vecs]
cases = [("cfg2_modes234", A, (2, 3, 4)), ("cfg2_modes123", A, (1, 2, 3)), ("cfg2_all4", A, (1, 2, 3, 4))]
T4, _ = W.cfg4()
A4 = tl.DenseTensor.from_memory(T4.shape, W.layout_buffer(T4, (1, 2, 3)))
del T4
u = tl.DenseTensor.from_memory((400,), np.full(400, 400 ** -0.5))
cases += [("cfg4_skip1", A4, (2, 3)), ("cfg4_skip3", A4, (1, 2)), ("cfg4_skip2", A4, (1, 3))]
for name, X, modes in cases:
    vs = [V[q - 1] if X is A else u for q in modes]
    row = {}
    for chain in ("1", "0"):
        os.environ["TL_TV_CHAIN"] = chain
        row["chain" if chain == "1" else "launches"] = round(med(lambda: tl.times_vectors(X, vs, list(modes))), 2)
    os.environ["TL_TV_CHAIN"] = "1"
    a = tl.times_vectors(X, vs, list(modes)).numpy()
    os.environ["TL_TV_CHAIN"] = "0"
    b = tl.times_vectors(X, vs, list(modes)).numpy()
    row["bit_identical"] = a.tobytes() == b.tobytes()
    res[name] = row
print(json.dumps(res))
