"""Per-layer phase clocks of the tensor-core kernel (development aid): run with
UFPGD_LIB pointing at a -DUFPGD_MMA_TIMING build (tools/ab_build.sh timing
-DUFPGD_MMA_TIMING); thread 0 of realization 5000 stamps layer 10 into W."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U

names = ["split", "s1 issue", "s1 wait", "s1 drain", "Bs build", "s2 issue", "s2 wait", "drain+prox"]
for cfg, n in ((2, 65536), (4, 16384), (5, 65536)):
    w = U.CONFIGS[cfg]
    Hd = torch.empty((n, w.M, w.K), dtype=torch.complex64, device="cuda")
    U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, n, w.K, w.M, out=Hd)
    lam, eta = w.layer_params()
    acc = np.zeros(8)
    for r in range(5):
        W = U.unfolded_forward(Hd, lam, eta, w.c)["W"]
        torch.cuda.synchronize()
        # the probe CTA (blockIdx 5000) writes its stamps into its thread 0's realization:
        # 5000 ((16,128), (32,256)) or 10000 (config 2: the pair's first realization)
        st = W[10000 if cfg == 2 else 5000].reshape(-1).view(torch.float32).view(torch.int64)[:16].cpu().numpy()
        acc += np.diff(st[:9].astype(np.float64))
        pacc = np.diff(st[9:16].astype(np.float64)) + (pacc if r else 0)
    acc /= 5
    print(f"cfg{cfg}: total {acc.sum():.0f} clk/layer: " + "  ".join(f"{a} {b:.0f}" for a, b in zip(names, acc)))
    pn = ["loads+amax", "smem H", "TMEM H", "W0/power", "layers", "W out"]
    print(f"cfg{cfg}: prologue/epilogue clk: " + "  ".join(f"{a} {b:.0f}" for a, b in zip(pn, pacc / 5)))
