"""Development check of the tcgen05 kernel (mma.cu): single-layer closed forms,
the tensor-core kernel against the CUDA-core tile kernel, CUDA-event timing,
PGD timing and the clock64 phase probe (parity against the FP64 oracle is in
tests/test_gpu_mma.py — tools/ never loads the oracle)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U


def run(H, lam, eta, c, w0_mode=0, W0=None, mma=True):
    U.set_option("tensor_cores", int(mma))
    Hd = torch.from_numpy(H).cuda()
    W0d = torch.from_numpy(W0).cuda() if W0 is not None else None
    out = U.unfolded_forward(Hd, lam, eta, c, w0_mode=w0_mode, W0=W0d, want_per_realization=True)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


def rel(a, b):
    B = a.shape[0]
    return np.linalg.norm((a - b).reshape(B, -1), axis=1) / np.maximum(np.linalg.norm(b.reshape(B, -1), axis=1), 1e-30)


def one_layer(K=32, M=256, B=4, seed=0):
    rng = np.random.default_rng(seed)
    H = ((rng.standard_normal((B, M, K)) + 1j * rng.standard_normal((B, M, K))) / np.sqrt(2)).astype(np.complex64)
    c = np.full(K, np.sqrt(10.0))
    eta = np.array([1 / 469.0]); lam = np.array([0.0])
    Hk = np.transpose(H, (0, 2, 1)).astype(np.complex128)  # [B][K][M]
    # a) W0 = 0: W1 = eta diag(c) H^*
    o = run(H, lam, eta, c)
    ref = eta[0] * c[None, :, None] * np.conj(Hk)
    r = rel(np.transpose(o["W"], (0, 2, 1)), ref)
    print(f"({K},{M}) L=1 W0=0: rel max {r.max():.3e}", flush=True)
    if r.max() > 1e-5:
        Wg = np.transpose(o["W"], (0, 2, 1))
        print("  sample got", Wg[0, :3, :3], "\n  want", ref[0, :3, :3])
    # b) W0 given: W1 = W0 - eta (W0 H^T - diag c) H^*
    W0 = ((rng.standard_normal((B, M, K)) + 1j * rng.standard_normal((B, M, K))) * 0.05).astype(np.complex64)
    o = run(H, lam, eta, c, w0_mode=2, W0=W0)
    W0k = np.transpose(W0, (0, 2, 1)).astype(np.complex128)
    X = W0k @ np.transpose(Hk, (0, 2, 1)) - np.diag(c)[None]
    ref = W0k - eta[0] * X @ np.conj(Hk)
    r = rel(np.transpose(o["W"], (0, 2, 1)), ref)
    print(f"({K},{M}) L=1 W0 given: rel max {r.max():.3e}", flush=True)
    if r.max() > 1e-5:
        Wg = np.transpose(o["W"], (0, 2, 1))
        d = np.abs(Wg - ref)[0]
        print("  err by user", np.round(d.max(1), 4))
        print("  err by antenna (first 16)", np.round(d.max(0)[:16], 4))
        print("  G got", (Wg - W0k)[0, :2, :4], "\n  G want", (ref - W0k)[0, :2, :4])


def check(cfg=4, n=256):
    """Tensor-core kernel vs the CUDA-core tile kernel on the same inputs (the
    oracle comparison lives in tests/test_gpu_mma.py)."""
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 0, n)
    lam, eta = w.layer_params()
    om = run(H, lam, eta, w.c)
    ot = run(H, lam, eta, w.c, mma=False)
    r = rel(om["W"], ot["W"].astype(np.complex128))
    print(f"cfg{cfg} n={n}: mma vs tile W rel max {r.max():.3e} median {np.median(r):.3e}; "
          f"diverged {int((om['diverged_at'] >= 0).sum())}; active {om['active'].mean():.1f}; "
          f"l21 rel {np.max(np.abs(om['l21'] - ot['l21']) / ot['l21']):.2e}", flush=True)


def timing(cfg=4, n=16384, reps=3):
    w = U.CONFIGS[cfg]
    Hd = torch.empty((n, w.M, w.K), dtype=torch.complex64, device="cuda")
    U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, n, w.K, w.M, out=Hd)
    lam, eta = w.layer_params()
    W = torch.empty_like(Hd)
    for mma in (True, False):
        U.set_option("tensor_cores", int(mma))
        U.unfolded_forward(Hd, lam, eta, w.c, out=W); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps): U.unfolded_forward(Hd, lam, eta, w.c, out=W)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        fl = w.flops_per_realization() * n
        print(f"{'mma ' if mma else 'tile'} cfg{cfg} B={n}: {ms:.3f} ms  {n / ms * 1e3 / 1e3:.1f} k/s  "
              f"{fl / ms / 1e9:.1f} TFLOP/s (FP32-equivalent)", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["one", "cfg4", "time"]
    if what[0] in ("phases", "pgd"):
        what = ["deferred"]
    if what[0] == "prof":  # one launch per config for ncu (-k regex:mma_kernel)
        for c in what[1:]:
            timing(int(c), 16384 if c == "4" else 65536, reps=1)
        sys.exit(0)
    if "one" in what:
        one_layer(32, 256)
        one_layer(16, 128)
    if "cfg4" in what: check(4)
    if "cfg5" in what: check(5, 1024)
    if "time" in what:
        timing(4, 16384)
        timing(5, 65536)


def pgd_timing(cfg, n=4096, iters=1000):
    """Fixed-step PGD (in-kernel 30-step power iteration) at the config's shape:
    tensor-core kernel vs the FFMA2 tile kernel."""
    w = U.CONFIGS[cfg]
    Hd = torch.empty((n, w.M, w.K), dtype=torch.complex64, device="cuda")
    U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, n, w.K, w.M, out=Hd)
    for mma in (True, False):
        U.set_option("tensor_cores", int(mma))
        U.pgd_fixed(Hd, 0.05, 10, w.c); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); U.pgd_fixed(Hd, 0.05, iters, w.c); e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        fl = iters * (16 * w.K * w.K * w.M + 10 * w.K * w.M) * n
        print(f"{'mma ' if mma else 'tile'} PGD-{iters} ({w.K},{w.M}) B={n}: {ms:.2f} ms  "
              f"{fl / ms / 1e9:.1f} TFLOP/s (FP32-equivalent)", flush=True)


def phase_probe(cfg):
    """With a -DUFPGD_MMA_TIMING library (tools/ab_build.sh): clock64 stamps of
    layer 10 of realization 5000, written into its W."""
    w = U.CONFIGS[cfg]
    n = 16384
    Hd = torch.empty((n, w.M, w.K), dtype=torch.complex64, device="cuda")
    U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, n, w.K, w.M, out=Hd)
    lam, eta = w.layer_params()
    W = torch.empty_like(Hd)
    for _ in range(2):
        U.unfolded_forward(Hd, lam, eta, w.c, out=W)
    torch.cuda.synchronize()
    t = W[5000].view(torch.int64).flatten()[:9].cpu().numpy()
    d = np.diff(t)
    names = ["Wop+sync", "s1 issue", "s1 wait", "E1+sync", "Bs+sync", "s2 issue", "s2 wait", "E2+prox"]
    print(f"cfg{cfg} layer clocks total {t[8] - t[0]}: " + ", ".join(f"{a} {b}" for a, b in zip(names, d)))


if __name__ == "__main__" and sys.argv[1:2] == ["phases"]:
    for c in sys.argv[2:]:
        phase_probe(int(c))
if __name__ == "__main__" and sys.argv[1:2] == ["pgd"]:
    for c in sys.argv[2:]:
        pgd_timing(int(c))
