"""Zero-padded fused path vs the general kernel on shapes without a
specialised kernel (development aid): ms per 65,536-realization batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U

B = 65536
for K, M in [(3, 10), (6, 48), (5, 40), (7, 64), (8, 50), (12, 100), (24, 200)]:
    H = U.generate_channels_device(1, 2, 10.0, 0, B, K, M)
    lam, eta = U.project_params(*U.layer_params(5, 20, K, M), K, M)
    c = np.full(K, np.sqrt(10.0))
    W = torch.empty_like(H)
    res = {}
    for mode in ("pad", "general"):
        if mode == "general":
            U.set_option("zero_pad", 0)
        run = lambda: U.unfolded_forward(H, lam, eta, c, w0_mode=U.W0_ZERO, out=W)
        run(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            run()
        b.record(); torch.cuda.synchronize()
        res[mode] = a.elapsed_time(b) / 5
        U.set_option("zero_pad", 1)
    fl = 20 * (16 * K * K * M + 10 * K * M) * B
    print(f"({K:2d},{M:3d})  padded {res['pad']:8.3f} ms ({fl / res['pad'] / 1e9:5.1f} useful TFLOP/s)   "
          f"general {res['general']:8.3f} ms ({fl / res['general'] / 1e9:5.1f})   x{res['general'] / res['pad']:.2f}", flush=True)
