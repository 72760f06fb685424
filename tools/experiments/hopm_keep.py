"""Config-4 HOPM sweeps/s (50 sweeps in one graph) and a hash of the lambda
history + vectors, under the environment's TL_HOPM_KEEP_MB (pass prefetch)."""
import hashlib, os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
import workloads as W
T, _ = W.cfg4()
A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3)))
del T
r = tl.HopmRunner(A, max_sweeps=50, tol=0.0)
r.launch(); torch.cuda.synchronize()
ts = []
for _ in range(7):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); r.launch(); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
st = r.state()
h = hashlib.sha256(np.asarray(st.lambda_history, dtype=np.float64).tobytes())
for v in st.u:
    h.update(np.asarray(v.numpy(), dtype=np.float64).tobytes())
print(json.dumps({"keep_mb": os.environ.get("TL_HOPM_KEEP_MB", "0"), "sweeps_per_s": round(50 / (min(ts) * 1e-3), 1),
                  "median_sweeps_per_s": round(50 / (sorted(ts)[3] * 1e-3), 1), "sha": h.hexdigest()[:16]}))
