"""Quick CUDA-event timing of the fused kernels (development aid, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U

def t_uf(cfg, reps=10, n=None):
    w = U.CONFIGS[cfg]
    if n is not None:
        import dataclasses
        w = dataclasses.replace(w, B=n)
    t0 = time.time(); H = U.make_inputs(w); tg = time.time() - t0
    lam, eta = w.layer_params()
    Hd = torch.from_numpy(H).cuda(); W = torch.empty_like(Hd)
    for _ in range(3): U.unfolded_forward(Hd, lam, eta, w.c, out=W)
    torch.cuda.synchronize()
    call = lambda: U.unfolded_forward(Hd, lam, eta, w.c, out=W)  # noqa: E731
    if os.environ.get("QT_GRAPH"):  # CUDA-graph replay: no host launch cost in the timing
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            U.unfolded_forward(Hd, lam, eta, w.c, out=W)
        call = g.replay
        reps = max(reps, 100)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(int(os.environ.get("QT_ROUNDS", "5"))):  # best of rounds: robust to box noise
        s.record()
        for _ in range(reps): call()
        e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / reps)
    ms = best
    fl = w.flops_per_realization() * w.B
    print(f"cfg{cfg} B={w.B}: {ms:.3f} ms/batch  {w.B/ms*1e3/1e6:.2f} M precoders/s  {fl/ms/1e9:.2f} TFLOP/s  (gen {tg:.1f}s)", flush=True)

def t_pgd(n=4096):
    w = U.CONFIGS[3]
    H = U.make_inputs(w, 0, n); Hd = torch.from_numpy(H).cuda()
    U.pgd_fixed(Hd, w.lambda_pgd, 100, w.c); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); U.pgd_fixed(Hd, w.lambda_pgd, w.L, w.c); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    fl = w.flops_per_realization() * n
    print(f"cfg3 B={n}: {ms:.3f} ms  {n/ms*1e3/1e3:.2f} k precoders/s  {fl/ms/1e9:.2f} TFLOP/s", flush=True)

def t_gen(cfg):
    w = U.CONFIGS[cfg]
    n = w.B if cfg != 5 else 65536
    Hd = torch.empty((n, w.M, w.K), dtype=torch.complex64, device="cuda")
    U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, n, w.K, w.M, out=Hd); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, n, w.K, w.M, out=Hd); e.record()
    torch.cuda.synchronize(); ms = s.elapsed_time(e)
    t0 = time.time(); U.make_inputs(w, 0, n); th = time.time() - t0
    print(f"gen cfg{cfg} B={n}: device {ms:.3f} ms ({n/ms*1e3/1e6:.2f} M realizations/s), host {th*1e3:.0f} ms", flush=True)

if __name__ == "__main__":
    if sys.argv[1:2] == ["gen"]:
        for c in (1, 2, 3, 4, 5): t_gen(c)
        sys.exit(0)
    for c in [int(x) for x in (sys.argv[1:] or ["1", "2", "4"])]:
        if c == 3: t_pgd()
        elif c == 5: t_uf(5, reps=2, n=int(os.environ.get("CFG5_B", "65536")))
        else: t_uf(c, reps=10 if c != 4 else 2)
