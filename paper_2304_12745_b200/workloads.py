"""BASELINE.json workloads as seeded synthetic inputs.

Common settings: SystemConfig::uniform(K, M, gamma = 10 (10 dB), sigma = 1,
alpha = 1) (commands.hpp:20-22), so c_k = sqrt(10). Channels are
generate_channel(Rng::stream(seed_h, i)) with per-user power gains
log-uniform over [-R, 0] dB, rounded once to complex64. Layer parameters
lambda_l ~ U[0.01, 0.1], mu_l ~ U[0.5, 1.5] / mp_bound from Rng::stream(seed_p,
0), then project_params (unfolded.cpp:71-81) because forward rejects
unprojected steps (unfolded.cpp:88). Seeds: seed_h = 1000 + config,
seed_g = seed_h ^ 0x6A1D, seed_p = seed_h ^ 0x9A4A.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import capi


def mp_bound(K: int, M: int) -> float:
    """pgd.cpp:111-118."""
    if K < 1 or M < 1:
        raise ValueError("mp_bound: dimensions must be positive")
    e = math.sqrt(K) + math.sqrt(M)
    return e * e


def project_params(lam, eta, K: int, M: int):
    """unfolded.cpp:71-81: lambda <- max(0, lambda); eta clamped to [1/(2L), 1/L]."""
    hi = 1.0 / mp_bound(K, M)
    lo = 0.5 * hi
    lam = np.maximum(0.0, np.asarray(lam, dtype=np.float64))
    eta = np.minimum(np.maximum(np.asarray(eta, dtype=np.float64), lo), hi)
    return lam, eta


@dataclass(frozen=True)
class Workload:
    config: int
    kind: str          # "unfolded" or "pgd"
    K: int
    M: int
    L: int             # layers or PGD iterations
    B: int
    gain_db: float
    w0_mode: int
    lambda_pgd: float = 0.05
    power_steps: int = 30

    @property
    def seed_h(self) -> int:
        return 1000 + self.config

    @property
    def seed_g(self) -> int:
        return self.seed_h ^ 0x6A1D

    @property
    def seed_p(self) -> int:
        return self.seed_h ^ 0x9A4A

    @property
    def c(self) -> np.ndarray:
        return np.full(self.K, math.sqrt(10.0))  # sigma_nu * sqrt(gamma), gamma = 10

    def layer_params(self):
        lam, eta = capi.layer_params(self.seed_p, self.L, self.K, self.M)
        return project_params(lam, eta, self.K, self.M)

    def name(self) -> str:
        if self.kind == "pgd":
            return f"cfg{self.config}: PGD-{self.L} (+{self.power_steps}-step power iteration), K={self.K}, M={self.M}, B={self.B}"
        return f"cfg{self.config}: UF-PGD-{self.L}, K={self.K}, M={self.M}, B={self.B}, gains {self.gain_db:g} dB"

    def flops_per_realization(self, exact_w0: bool = True) -> float:
        """SURVEY §8d cost model: L (16 K^2 M + 10 K M) (+ power steps).
        exact_w0: with W0 = 0 the kernels compute neither layer-0 contraction
        (W0 H^T is identically zero and X' = -diag(c) makes the second a
        per-entry scaling), so 2L - 2 contractions are counted, not 2L."""
        K, M, L = self.K, self.M, self.L
        contractions = 2 * L - (2 if (exact_w0 and self.w0_mode == capi.W0_ZERO) else 0)
        f = contractions * 8 * K * K * M + L * 10 * K * M
        if self.kind == "pgd":
            f += self.power_steps * (16 * K * M + 14 * M)
        return float(f)

    def tensor_flops_per_realization(self):
        """Tensor-core flops the tcgen05 kernel (csrc/mma.cu) issues per
        realization at (16,128) / (32,256) unfolded — and at (8,64), where two
        realizations share a (16,128) frame with their own MMAs — None elsewhere: stage 1
        2 Q (2R) M per layer (Q = 4K rows [W_hi; W_lo], N = [H_hi | H_lo]),
        skipped at a W0 = 0 layer 0; stage 2 (M/128) 2*128 (2R R + R R) per
        layer (H_hi [Bs_hi | Bs_lo] + H_lo Bs_hi), R = 2K. The 3-term f16
        split performs ~3x the FP32-equivalent work."""
        if self.kind != "unfolded" or (self.K, self.M) not in ((8, 64), (16, 128), (32, 256)):
            return None
        K, M, L = self.K, self.M, self.L
        n1 = L - 1 if self.w0_mode == capi.W0_ZERO else L
        if (K, M) == (8, 64):
            # realization pairs in the (16,128) frame, each with its own MMAs:
            # stage 1 one M = 64 (the pair's [W_hi; W_lo] rows), N = 32, K = 64
            # chain; stage 2 one K = 16 step, M = 128, N = 32 + 16
            return n1 * 2.0 * 64 * 32 * 64 + L * 2.0 * 128 * 48 * 16
        R, Q = 2 * K, 4 * K
        s1 = 2.0 * Q * (2 * R) * M
        s2 = (M // 128) * 2.0 * 128 * 3 * R * R
        return n1 * s1 + L * s2

    def bytes_per_realization(self) -> float:
        return 16.0 * self.K * self.M  # H in + W out, complex64


CONFIGS = {
    1: Workload(1, "unfolded", 4, 32, 20, 1024, 0.0, capi.W0_ZERO),
    2: Workload(2, "unfolded", 8, 64, 20, 65536, 20.0, capi.W0_ZERO),
    3: Workload(3, "pgd", 8, 64, 5000, 4096, 0.0, capi.W0_CONJ_H),
    4: Workload(4, "unfolded", 32, 256, 20, 16384, 30.0, capi.W0_ZERO),
    5: Workload(5, "unfolded", 16, 128, 20, 1048576, 30.0, capi.W0_ZERO),
}


def make_inputs(w: Workload, first_index: int = 0, B: int | None = None, threads: int = 0) -> np.ndarray:
    """Host complex64 channels [B, M, K] for realizations first_index..+B."""
    n = w.B if B is None else B
    return capi.generate_channels(w.seed_h, w.seed_g, w.gain_db, first_index, n, w.K, w.M, threads)
