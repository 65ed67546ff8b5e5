"""PGD with residual_tol: the fused team kernel's early exit vs the general
kernel (development aid): config 3's 4,096 (8,64) channels, lambda 0.05."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U

w = U.CONFIGS[3]
H = torch.from_numpy(U.make_inputs(w)).cuda()
for tol in (1e-4, 1e-5, 0.0):
    U.pgd_fixed(H, w.lambda_pgd, 5000, w.c, residual_tol=tol)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = U.pgd_fixed(H, w.lambda_pgd, 5000, w.c, residual_tol=tol, want_per_realization=True)
    b.record(); torch.cuda.synchronize()
    its = out["iterations"].cpu().numpy()
    print(f"residual_tol {tol:g}: {a.elapsed_time(b):8.2f} ms, iterations mean {its.mean():.0f} max {its.max()}", flush=True)
