"""A/B for the verdict's question "does the tensor path win at K = 8?"
(development aid, result quoted in DESIGN.md §9): config 2's (8,64)
realizations run in block-diagonal pairs on the tcgen05 (16,128) kernel —
exact for the unfolded PGD (X = W H^T, X' H^* and the per-antenna prox never
mix the two diagonal blocks; c_pair = [c; c], W0 = 0) — against the FFMA2
team kernel on the same batch, CUDA-event timed, with the outputs compared."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_12745_b200 as U

w = U.CONFIGS[2]
B = w.B
H = U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, B, w.K, w.M)
lam, eta = w.layer_params()
c = w.c


def pairs(H):  # [B][64][8] -> block-diagonal [B/2][128][16]
    P = torch.zeros((B // 2, 2 * w.M, 2 * w.K), dtype=H.dtype, device=H.device)
    P[:, :w.M, :w.K] = H[0::2]
    P[:, w.M:, w.K:] = H[1::2]
    return P.contiguous()


Hp = pairs(H)
cp = np.concatenate([c, c])


def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = fn()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best, out


Wt = torch.empty_like(H)
Wp = torch.empty_like(Hp)
t_team, o_team = timeit(lambda: U.unfolded_forward(H, lam, eta, c, out=Wt))
t_mma, o_mma = timeit(lambda: U.unfolded_forward(Hp, lam, eta, cp, out=Wp))
W_from_pairs = torch.empty_like(H)
W_from_pairs[0::2] = Wp[:, :w.M, :w.K]
W_from_pairs[1::2] = Wp[:, w.M:, w.K:]
offdiag = max(Wp[:, :w.M, w.K:].abs().max().item(), Wp[:, w.M:, :w.K].abs().max().item())
d = (W_from_pairs - Wt).abs().flatten(1).norm(dim=1) / Wt.abs().flatten(1).norm(dim=1)
print(f"config 2, B = {B}: FFMA2 team kernel {t_team:.3f} ms ({B / t_team / 1e3:.2f} M/s); "
      f"tcgen05 (16,128) kernel on block-diagonal pairs {t_mma:.3f} ms ({B / t_mma / 1e3:.2f} M/s); "
      f"ratio {t_mma / t_team:.2f}x; off-diagonal max {offdiag:.1e}; W rel diff max {d.max().item():.2e}")
