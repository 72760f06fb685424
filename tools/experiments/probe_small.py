"""Device time of the small (L2-resident) ttvs inside HOPM, in isolation."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np
import torch

import paper_1711_10912_b200 as tl
from probe_ops import timeit

rng = np.random.default_rng(0)
for n in (400, 128, 1000):
    T = tl.DenseTensor.from_memory((n, n), rng.standard_normal(n * n))
    u = tl.DenseTensor.from_memory((n,), rng.standard_normal(n))
    for mode in (1, 2):
        med, mn = timeit(lambda: tl.ttv(T, u, mode), reps=20)
        print(f"ttv {n}x{n} mode {mode}: {med * 1e3:.2f} us (min {mn * 1e3:.2f})", flush=True)
# a 3-D small one: 400x400x4
T3 = tl.DenseTensor.from_memory((400, 400, 4), rng.standard_normal(400 * 400 * 4))
u4 = tl.DenseTensor.from_memory((4,), rng.standard_normal(4))
med, _ = timeit(lambda: tl.ttv(T3, u4, 3), reps=20)
print(f"ttv 400x400x4 mode 3: {med * 1e3:.2f} us")
