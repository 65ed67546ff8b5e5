"""oracle_solve at scale timing: FP64 device path vs the
FP64 oracle on the host cores (development aid)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2304_12745_b200 as U
from oracle import oracle as O

K, M, lam = 8, 64, 1.0 / 15.0
c = np.full(K, math.sqrt(10.0))
for B in (256, 2048):
    H = U.generate_channels_device(33, 0, 0.0, 0, B, K, M, dtype=torch.complex128)
    U.oracle_solve(H[:8].contiguous(), c, lam)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = U.oracle_solve(H, c, lam)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    its = out["iterations"].cpu().numpy()
    print(f"device oracle_solve B={B}: {dt:.2f} s, {B / dt:.1f} channels/s, iterations mean {its.mean():.0f} max {its.max()}",
          flush=True)
Hh = U.generate_channels_device(33, 0, 0.0, 0, 16, K, M, dtype=torch.complex128).cpu().numpy()
cfg = O.SystemConfig.uniform(K, M, 10.0)
t0 = time.perf_counter()
for b in range(4):
    O.oracle_solve(O.from_storage(Hh[b], K, M), cfg, lam)
dt = time.perf_counter() - t0
print(f"host oracle (1 thread, FP64): {4 / dt:.2f} channels/s", flush=True)
