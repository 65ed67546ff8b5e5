"""Host cost of one unfolded_forward call (ctypes + validation + launches),
measured on config 1 whose kernel is ~16 us (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_12745_b200 as U

w = U.CONFIGS[1]
H = torch.from_numpy(U.make_inputs(w)).cuda()
lam, eta = w.layer_params()
W = torch.empty_like(H)
for _ in range(20):
    U.unfolded_forward(H, lam, eta, w.c, out=W)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    U.unfolded_forward(H, lam, eta, w.c, out=W)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host per call {1e6 * (t1 - t0) / n:.1f} us (enqueue only), with drain {1e6 * (time.perf_counter() - t0) / n:.1f} us")
