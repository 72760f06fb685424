"""HOPM on the config-4 tensor stored in every permutation layout: sweeps/s and the lambda history against the
first-order run (the result is layout-independent: every ttv output is the same k-ordered fold)."""
import itertools, json, os, sys
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import torch
import paper_1711_10912_b200 as tl
import workloads as W
T, _ = W.cfg4()
ref = None
for lay in itertools.permutations((1, 2, 3)):
    A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, lay), layout=lay)
    r = tl.HopmRunner(A, max_sweeps=50, tol=0.0)
    r.launch(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); r.launch(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    st = r.state()
    if ref is None:
        ref = st.lambda_history
    print(json.dumps({"layout": lay, "sweeps_per_s": round(50 / (min(ts) * 1e-3), 1), "lambda50": st.lambda_history[-1],
                      "history_equals_first_order": st.lambda_history == ref}), flush=True)
    r.close(); del A, r
    torch.cuda.empty_cache()
