"""Times ufpgd_gpu_layers_general (the taped forward, unfolded.hpp:40-62) at
config 2 — no tapes, iterates only, iterates + tape — with CUDA events, and
prints the bytes each variant writes (development aid; UFPGD_LIB selects an
A/B build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2304_12745_b200 as U

w = U.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
B = int(sys.argv[2]) if len(sys.argv) > 2 else w.B
K, M, L = w.K, w.M, w.L
H = U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, B, K, M)
lam, eta = w.layer_params()
thr = lam * eta
def fused(tc):
    with U.options(tensor_cores=tc):
        return U.unfolded_forward(H, lam, eta, w.c, w0_mode=U.W0_CONJ_H)


for name, kw in (("fused team (untaped)", None), ("fused tcgen05 (untaped)", 1), ("plain", {}), ("iterates", dict(iterates=True)), ("tape+iterates", dict(iterates=True, tape=True))):
    if isinstance(kw, dict):
        fn = lambda kw=kw: U.layers_general(H, eta, thr, w.c, **kw)
    else:
        fn = lambda tc=kw or 0: fused(tc)
        kw = {}
    r = fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    wr = 16 * K * M  # H in + W out
    if kw.get("iterates"):
        wr += (L + 1) * 8 * K * M
    if kw.get("tape"):
        wr += L * (8 * K * M + 8 * M)
    print(f"cfg{w.config} B={B} {name}: {best:.3f} ms  {B / best / 1e3:.2f} M/s  "
          f"{wr * B / best / 1e6:.0f} GB/s moved", flush=True)
    del r
