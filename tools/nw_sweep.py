"""Warps-per-block sweep of the team kernel over batch sizes (development aid):
UFPGD_FUSED_WARPS is read per launch."""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_12745_b200 as U

for cfg, sizes in ((2, (8192, 16384, 32768, 65536, 262144)), (1, (1024, 16384, 65536))):
    for n in sizes:
        w = dataclasses.replace(U.CONFIGS[cfg], B=n)
        H = torch.from_numpy(U.make_inputs(w)).cuda(); W = torch.empty_like(H)
        lam, eta = w.layer_params()
        row = []
        for nw in (1, 2, 4, 8):
            U.set_option("fused_warps", nw)
            for _ in range(3): U.unfolded_forward(H, lam, eta, w.c, out=W)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            reps = max(3, int(2e5 / n))
            for _ in range(5):
                s.record()
                for _ in range(reps): U.unfolded_forward(H, lam, eta, w.c, out=W)
                e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e) / reps)
            row.append(f"nw={nw}: {best*1e3:8.1f} us")
        U.set_option("fused_warps", 0)
        print(f"cfg{cfg} B={n:7d}  " + "  ".join(row), flush=True)
