"""Representative slow ttv cases found by layout_sweep.py (tiny or huge
contracted extents, permuted outputs), plus the config-5 layouts as a
regression guard: time (graph replays), fraction of the HBM peak, regime,
and a sha of the output (bit-exactness across kernel changes).

    python tools/experiments/ttv_cases.py
"""
import ctypes
import hashlib
import json
import os
import sys

import torch

R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [R, os.path.join(R, "tests"), os.path.join(R, "tools", "experiments")]
import paper_1711_10912_b200 as tl  # noqa: E402
from paper_1711_10912_b200.layout import TensorMeta  # noqa: E402
from sweep_ttm5 import timeit  # noqa: E402

CASES = [
    ("a", torch.float64, (237, 10, 2, 11277), (3, 1, 4, 2), 3),
    ("b", torch.float32, (2, 318, 4, 72, 15, 6, 7), (6, 5, 2, 1, 7, 3, 4), 6),
    ("c", torch.float32, (2, 5, 4305, 56, 6, 9), (5, 4, 3, 1, 2, 6), 1),
    ("d", torch.float32, (7, 3, 6, 3, 20, 36, 551), (3, 5, 1, 4, 7, 6, 2), 4),
    ("e", torch.float32, (6, 29, 7, 11, 2, 634, 10), (7, 5, 3, 6, 1, 2, 4), 5),
    ("f", torch.float64, (1848, 2, 21263), (2, 1, 3), 2),
    ("g", torch.float32, (5, 4, 532, 801, 2, 8), (2, 6, 4, 3, 5, 1), 2),
    ("h", torch.float32, (2, 5, 4305, 56, 6, 9), (5, 4, 3, 1, 2, 6), 3),
    ("i", torch.float64, (201, 333367), (2, 1), 2),
    ("j", torch.float32, (189286, 709), (2, 1), 1),
    ("k", torch.float64, (15, 42, 2, 4, 22, 5, 147), (5, 1, 2, 3, 7, 6, 4), 3),
    ("cfg5s0", torch.float64, (3, 33, 5, 17, 9, 2, 640), (5, 3, 2, 1, 6, 4, 7), 5),
    ("cfg5s5", torch.float64, (3, 33, 5, 17, 9, 2, 640), (7, 4, 2, 1, 6, 3, 5), 5),
]


def peak():
    try:
        return float(json.load(open(os.path.join(R, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6545.6


def main():
    only = set(sys.argv[1:])
    pk = peak()
    L = tl._abi.lib()
    g = torch.Generator(device="cuda")
    for name, dtype, shape, layout, mode in CASES:
        if only and name not in only:
            continue
        g.manual_seed(len(name) + sum(shape))
        n = 1
        for e in shape:
            n *= e
        s = 4 if dtype == torch.float32 else 8
        buf = torch.rand(n, dtype=dtype, device="cuda", generator=g)
        A = tl.DenseTensor._wrap(TensorMeta(shape, layout=layout), buf)
        v = tl.DenseTensor._wrap(TensorMeta((shape[mode - 1],)), torch.rand(shape[mode - 1], dtype=dtype, device="cuda", generator=g))
        C = tl.ttv(A, v, mode)
        sha = hashlib.sha256(C.buffer.cpu().numpy().tobytes()).hexdigest()[:12]
        us = timeit(lambda: tl.ttv(A, v, mode), n=5)
        nbytes = s * (n + shape[mode - 1] + n // shape[mode - 1])
        info = ctypes.create_string_buffer(512)
        L.tl_plan_describe(0, A.desc(), None, mode, info, 512)
        d = json.loads(info.value.decode())
        print(json.dumps({"case": name, "us": round(us, 1), "frac": round(nbytes / us / 1e3 / pk, 3), "sha": sha,
                          "regime": d.get("regime"), "O": d.get("O"), "K": d.get("K"), "I": d.get("I"),
                          "ident": d.get("ident")}), flush=True)
        del A, buf, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
