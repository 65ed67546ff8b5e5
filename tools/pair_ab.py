"""Config 2 on the tcgen05 realization-pair kernel vs the FFMA2 team kernel
(ufpgd_gpu_set_option(UFPGD_OPT_TENSOR_CORES, 0)): CUDA-graph timing, outputs
compared (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_12745_b200 as U

w = U.CONFIGS[2]
B = int(sys.argv[1]) if len(sys.argv) > 1 else w.B
H = U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, B, w.K, w.M)
lam, eta = w.layer_params()


def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


res = {}
for tc in (1, 0):
    U.set_option("tensor_cores", tc)
    W = torch.empty_like(H)
    t = timeit(lambda: U.unfolded_forward(H, lam, eta, w.c, out=W))
    res[tc] = (t, W.clone())
    print(f"tensor cores {tc}: {t:.3f} ms ({B / t / 1e3:.2f} M/s)", flush=True)
U.set_option("tensor_cores", 1)
d = (res[1][1] - res[0][1]).abs().flatten(1).norm(dim=1) / res[0][1].abs().flatten(1).norm(dim=1).clamp_min(1e-30)
print(f"pair vs team: W rel diff max {d.max().item():.2e} median {d.median().item():.2e}; ratio {res[1][0] / res[0][0]:.3f}")

if len(sys.argv) > 2 and sys.argv[2] == "pgd":  # config 3: PGD-5000 (+ in-kernel 30-step power iteration)
    w3 = U.CONFIGS[3]
    H3 = U.generate_channels_device(w3.seed_h, w3.seed_g, w3.gain_db, 0, w3.B, w3.K, w3.M)
    r3 = {}
    for tc in (1, 0):
        U.set_option("tensor_cores", tc)
        t = timeit(lambda: U.pgd_fixed(H3, w3.lambda_pgd, w3.L, w3.c), reps=2)
        r3[tc] = (t, U.pgd_fixed(H3, w3.lambda_pgd, w3.L, w3.c)["W"].clone())
        print(f"cfg3 tensor cores {tc}: {t:.3f} ms", flush=True)
    U.set_option("tensor_cores", 1)
    d = (r3[1][1] - r3[0][1]).abs().flatten(1).norm(dim=1) / r3[0][1].abs().flatten(1).norm(dim=1).clamp_min(1e-30)
    print(f"cfg3 pair vs team: W rel diff max {d.max().item():.2e} median {d.median().item():.2e}; "
          f"ratio {r3[1][0] / r3[0][0]:.3f}")

if len(sys.argv) > 2 and sys.argv[2] == "tol":  # config 3's data with solve_pgd's residual_tol = 1e-4
    w3 = U.CONFIGS[3]
    H3 = U.generate_channels_device(w3.seed_h, w3.seed_g, w3.gain_db, 0, w3.B, w3.K, w3.M)
    r3 = {}
    for tc in (1, 0):
        U.set_option("tensor_cores", tc)
        t = timeit(lambda: U.pgd_fixed(H3, w3.lambda_pgd, w3.L, w3.c, residual_tol=1e-4), reps=2)
        o = U.pgd_fixed(H3, w3.lambda_pgd, w3.L, w3.c, residual_tol=1e-4)
        r3[tc] = (t, o["W"].clone(), o["iterations"].cpu().numpy())
        print(f"cfg3 tol 1e-4 tensor cores {tc}: {t:.3f} ms, mean iterations {r3[tc][2].mean():.0f}", flush=True)
    U.set_option("tensor_cores", 1)
    import numpy as np
    print(f"iterations |pair - team| max {np.abs(r3[1][2] - r3[0][2]).max()}, ratio {r3[1][0] / r3[0][0]:.3f}")
