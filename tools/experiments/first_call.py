"""Where the first hot-path call of a process spends its time (acceptance c2)."""
import time
import torch
t0 = time.perf_counter()
import paper_1711_10912_b200 as tl
from paper_1711_10912_b200 import _abi
t1 = time.perf_counter()
a = tl.DenseTensor((4, 2, 3))
torch.cuda.synchronize()
t2 = time.perf_counter()
_abi.lib(); t3 = time.perf_counter()
_abi.lib().tl_device_arch(); t4 = time.perf_counter()
for j in range(a.size):
    a.set_memory(j, j)
t5 = time.perf_counter()
v = a.view(tl.Range(1, 2, 3), tl.Range(0, 1, 1), 2)
m = v.materialize(); t6 = time.perf_counter()
m2 = v.materialize(); t7 = time.perf_counter()
print(f"import {1e3*(t1-t0):.1f} ms, first tensor {1e3*(t2-t1):.1f}, lib load {1e3*(t3-t2):.2f}, arch {1e3*(t4-t3):.2f}, "
      f"set_memory x24 {1e3*(t5-t4):.2f}, first materialize {1e3*(t6-t5):.2f}, second {1e3*(t7-t6):.3f} ms")
