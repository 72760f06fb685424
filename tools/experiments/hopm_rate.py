import os, sys, json, time
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import torch
import paper_1711_10912_b200 as tl
import workloads as W
T, _ = W.cfg4()
A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3)))
r = tl.HopmRunner(A, max_sweeps=50, tol=0.0)
r.launch(); torch.cuda.synchronize()
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); r.launch(); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
st = r.state()
print(json.dumps({"sweeps_per_s": round(50 / (min(ts) * 1e-3), 1), "lambda": st.lambda_history[-1]}))
