"""Zero-copy probe: the fused kernel reading H from / writing W to pinned host
memory directly (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U
from paper_2304_12745_b200.capi import lib, _f64, _ptr

w = U.CONFIGS[2]
Hh = torch.from_numpy(U.make_inputs(w)).pin_memory()
Wh = torch.empty_like(Hh).pin_memory()
lam, et, cc = _f64(w.layer_params()[0]), _f64(w.layer_params()[1]), _f64(w.c)
div = torch.empty(w.B, dtype=torch.int32, device="cuda")
stats = torch.empty(3, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run():
    rc = lib().ufpgd_gpu_unfolded_forward(Hh.data_ptr(), w.B, w.K, w.M, _ptr(lam), _ptr(et), lam.size, _ptr(cc),
                                          w.w0_mode, None, Wh.data_ptr(), div.data_ptr(), None, None,
                                          stats.data_ptr(), 1.0, 0, s)
    assert rc == 0, rc
for _ in range(2): run()
torch.cuda.synchronize()
best = 0
for _ in range(3):
    t0 = time.perf_counter()
    for _ in range(10):
        run(); st = stats.cpu()
    torch.cuda.synchronize()
    best = max(best, 10 * w.B / (time.perf_counter() - t0))
print(f"zero-copy e2e: {best/1e6:.2f} M precoders/s")
ref = U.unfolded_forward(Hh.cuda(), *w.layer_params(), w.c, w0_mode=w.w0_mode)["W"].cpu()
print("identical to device path:", torch.equal(ref, Wh))
