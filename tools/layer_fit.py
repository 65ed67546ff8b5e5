import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2304_12745_b200 as U
for cfg in (4, 5):
    w = U.CONFIGS[cfg]
    n = 16384 if cfg == 4 else 65536
    Hd = torch.empty((n, w.M, w.K), dtype=torch.complex64, device="cuda")
    U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, n, w.K, w.M, out=Hd)
    lam, eta = w.layer_params()
    W = torch.empty_like(Hd)
    res = []
    for L in (1, 2, 5, 10, 20):
        l, e = lam[:L], eta[:L]
        U.unfolded_forward(Hd, l, e, w.c, out=W); torch.cuda.synchronize()
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3): U.unfolded_forward(Hd, l, e, w.c, out=W)
        t.record(); torch.cuda.synchronize()
        res.append((L, s.elapsed_time(t) / 3))
    Ls = np.array([r[0] for r in res]); ts = np.array([r[1] for r in res])
    b, a = np.polyfit(Ls[1:], ts[1:], 1)
    print(f"cfg{cfg}: " + ", ".join(f"L={L}: {t:.3f} ms" for L, t in res) + f"  fit (L>=2): {a:.3f} ms + {b:.4f} ms/layer", flush=True)
