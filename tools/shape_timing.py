"""Throughput of the fused team kernels on the BASELINE-neighbour shapes vs the
general kernel (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U

for K, M in ((4, 16), (4, 32), (4, 64), (8, 32), (8, 64), (8, 128), (6, 48)):
    B = 65536
    H = U.generate_channels_device(7, 0, 0.0, 0, B, K, M)
    lam, eta = U.project_params(*U.layer_params(3, 20, K, M), K, M)
    c = np.full(K, np.sqrt(10.0))
    W = torch.empty_like(H)
    run = lambda: U.unfolded_forward(H, lam, eta, c, out=W)
    run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # replay: no host launch overhead in the timing
    with torch.cuda.graph(g): run()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): g.replay()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    fl = (2 * 20 - 2) * 8 * K * K * M + 10 * K * M * 20
    print(f"({K},{M}) B={B}: {ms:.3f} ms  {B/ms/1e3:.2f} M/s  {fl*B/ms/1e9:.1f} TFLOP/s", flush=True)
