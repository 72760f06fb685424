"""Per-launch times of the cfg2 step's 12 ttvs in sequence (events on the
launch stream), under the environment's TL_TTV_KEEP_MB."""
import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import torch
import paper_1711_10912_b200 as tl
import workloads as W
T, vecs, T2 = W.cfg2()
vs = [tl.DenseTensor.from_memory((128,), v) for v in vecs]
A = {n: tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, l), layout=l) for n, l in W.CFG2_LAYOUTS.items()}
del T, T2
seq = [(n, m) for n in A for m in (1, 2, 3, 4)]
tot = {k: [] for k in seq}
for it in range(6):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)]
    ev[0].record()
    for i, (n, m) in enumerate(seq):
        tl.ttv(A[n], vs[m - 1], m)
        ev[i + 1].record()
    torch.cuda.synchronize()
    if it >= 2:
        for i, k in enumerate(seq):
            tot[k].append(ev[i].elapsed_time(ev[i + 1]) * 1e3)
out = {f"{n}_q{m}": round(sorted(v)[len(v) // 2], 1) for (n, m), v in tot.items()}
out["sum"] = round(sum(out.values()), 1)
print(os.environ.get("TL_TTV_KEEP_MB", "0"), json.dumps(out))
