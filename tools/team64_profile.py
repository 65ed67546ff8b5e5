"""One launch of the FP64 warp-per-realization PGD kernel for ncu (development aid)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U
K, M = 8, 64
H = U.generate_channels_device(33, 0, 0.0, 0, 8192, K, M, dtype=torch.complex128)
out = U.oracle_solve(H, np.full(K, math.sqrt(10.0)), 1 / 15, max_iters=2000)
torch.cuda.synchronize()
print("iterations mean", out["iterations"].float().mean().item())
