"""FP64 CPU oracle for the ufpgd hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module. The product package
(``paper_2304_12745_b200``) never imports it.

This is a ctypes wrapper over ``oracle/_build/libufpgd_oracle.so`` (the C++
restatement in ``ufpgd_oracle.cpp``) plus a Python mirror of the reference's
C++ API (``/root/reference/proj/core/include/ufpgd/*.hpp``) so the oracle tests
read like the reference's doctest suites. Matrices are numpy complex128 arrays
of shape (K, M) — row k = user, column m = antenna (``types.hpp:14-20``).

The random source ``Rng`` is restated a second time here in pure Python
(``std::mt19937_64`` + ``rng.cpp:9-40``) so the C++ restatement can be checked
against an independent one.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libufpgd_oracle.so")

ORA_OK, ORA_EINVAL, ORA_EDIVERGED, ORA_ECONVERGENCE, ORA_ESINGULAR = 0, -1, -3, -4, -5


def build() -> str:
    """Compile the oracle with its Makefile (g++ only, no CUDA)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        d, i, l, u64, i64 = C.c_double, C.c_int, C.c_long, C.c_uint64, C.c_int64
        P = C.c_void_p
        sigs = {
            "ora_default_thread_count": (i, []),
            "ora_mp_bound": (i, [i, i, P]),
            "ora_rng_draw": (i, [u64, u64, i, i, i, P, P]),
            "ora_generate_channel": (i, [u64, u64, i, i, i, P]),
            "ora_power_v0": (i, [i, P]),
            "ora_generate_channels_batch_f32": (i, [u64, u64, d, i64, i64, i, i, P, i]),
            "ora_layer_params": (i, [u64, i, i, i, P, P]),
            "ora_prox_l21": (i, [P, i, i, d, P]),
            "ora_grad_f": (i, [P, P, P, i, i, P]),
            "ora_pgd_step": (i, [P, P, P, i, i, d, d, P]),
            "ora_lipschitz": (i, [P, i, i, i, P]),
            "ora_l21_norm": (d, [P, i, i]),
            "ora_active_columns": (i, [P, i, i]),
            "ora_constraint_residual": (d, [P, P, P, i, i]),
            "ora_lagrangian": (d, [P, P, P, i, i, d]),
            "ora_zf_precoder": (i, [P, P, i, i, P]),
            "ora_forward": (i, [P, P, i, i, P, P, i, P, P, P, P, P, P, P, P]),
            "ora_solve_pgd": (i, [P, P, i, i, d, d, l, d, P, P, P, P]),
            "ora_forward_batch_f32": (i, [P, i64, P, i, i, P, P, i, i, P, P, P, P, P, P, i]),
            "ora_pgd_batch_f32": (i, [P, i64, P, i, i, d, P, l, d, i, P, P, P, P, P, P, P, i]),
            "ora_power_iteration_batch_f32": (i, [P, i64, i, i, i, P, P, i]),
            "ora_lagrangian_batch_f32": (i, [P, P, i64, P, i, i, d, P, i]),
            "ora_lagrangian_batch_f64": (i, [P, P, i64, P, i, i, d, P, i]),
            "ora_metrics": (i, [P, P, P, d, d, i, i, P]),
            "ora_backward": (i, [P, i, i, P, P, i, P, P, P, P, P, P, P]),
            "ora_train_sample": (i, [P, P, i, i, P, P, i, i, d, P, P, P]),
            "ora_train_batch_f32": (i, [P, i64, P, i, i, P, P, i, i, d, P, P, P, P, i]),
            "ora_metrics_batch_f32": (i, [P, P, i64, P, d, d, i, i, P, i]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


_KEEP: list = []


def _p(a: Optional[np.ndarray]):
    """Pointer to an array's data. Temporaries passed here are kept alive
    until the next top-level wrapper call (ctypes does not hold them)."""
    if a is None:
        return None
    _KEEP.append(a)
    if len(_KEEP) > 64:
        del _KEEP[:-32]
    return a.ctypes.data


# --------------------------------------------------------------------------
# errors.hpp:8-39
# --------------------------------------------------------------------------
class DivergenceError(RuntimeError):
    def __init__(self, what: str, index: int):
        super().__init__(what)
        self.index = index


class ConvergenceError(RuntimeError):
    pass


class SingularChannelError(RuntimeError):
    pass


class TrainingError(RuntimeError):
    pass


# --------------------------------------------------------------------------
# Storage helpers: (K, M) complex <-> interleaved [M][K] doubles
# --------------------------------------------------------------------------
def to_storage(A: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(A, dtype=np.complex128).T)


def from_storage(S: np.ndarray, K: int, M: int) -> np.ndarray:
    return np.ascontiguousarray(S.reshape(M, K).T)


# --------------------------------------------------------------------------
# rng.cpp:9-40 restated in pure Python (independent of the C++ restatement)
# --------------------------------------------------------------------------
_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 ([rand.predef]: 10000th output for seed 5489 is
    9981545732273789042)."""

    n, m = 312, 156

    def __init__(self, seed: int):
        self.mt = [0] * self.n
        self.mt[0] = seed & _MASK64
        for i in range(1, self.n):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK64
        self.idx = self.n

    def _twist(self):
        mt, n, m = self.mt, self.n, self.m
        upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
        for i in range(n):
            x = (mt[i] & upper) | (mt[(i + 1) % n] & lower)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + m) % n] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.n:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64


def mix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


class Rng:
    def __init__(self, seed: int):
        self.gen = MT19937_64(seed)

    @staticmethod
    def stream(seed: int, stream_index: int) -> "Rng":
        return Rng(mix64((seed ^ mix64(stream_index)) & _MASK64))

    def next_u64(self) -> int:
        return self.gen()

    def uniform(self) -> float:
        return float(self.gen() >> 11) * 2.0 ** -53

    def uniform_open(self) -> float:
        return float((self.gen() >> 11) + 1) * 2.0 ** -53

    def index_below(self, n: int) -> int:
        return self.gen() % n

    def complex_gaussian(self) -> complex:
        radius = math.sqrt(-math.log(self.uniform_open()))
        angle = 2.0 * math.pi * self.uniform()
        return complex(radius * math.cos(angle), radius * math.sin(angle))


def random_matrix(rows: int, cols: int, rng: Rng) -> np.ndarray:
    """support.hpp:87-94 (row-major draws)."""
    out = np.empty((rows, cols), dtype=np.complex128)
    for r in range(rows):
        for c in range(cols):
            out[r, c] = rng.complex_gaussian()
    return out


# --------------------------------------------------------------------------
# system_config.hpp / system_config.cpp
# --------------------------------------------------------------------------
@dataclass
class SystemConfig:
    K: int = 0
    M: int = 0
    sigma_nu: float = 1.0
    gamma: np.ndarray = field(default_factory=lambda: np.zeros(0))
    alpha: float = 1.0

    @staticmethod
    def uniform(num_users, num_antennas, sinr_target, noise_std=1.0, pa_scale=1.0):
        cfg = SystemConfig(num_users, num_antennas, noise_std,
                           np.full(max(num_users, 0), float(sinr_target)), pa_scale)
        cfg.validate()
        return cfg

    def validate(self):  # system_config.cpp:22-43
        if self.K < 1:
            raise ValueError("SystemConfig: K must be >= 1")
        if self.M < self.K:
            raise ValueError("SystemConfig: need K <= M")
        if not (self.sigma_nu >= 0.0):
            raise ValueError("SystemConfig: sigma_nu must be >= 0")
        g = np.asarray(self.gamma, dtype=np.float64)
        if g.shape != (self.K,):
            raise ValueError("SystemConfig: gamma must have K entries")
        if not np.all(g > 0.0):
            raise ValueError("SystemConfig: gamma must be > 0")
        if not (self.alpha > 0.0):
            raise ValueError("SystemConfig: alpha must be > 0")

    def constraint_diag(self) -> np.ndarray:  # system_config.cpp:45-47
        return self.sigma_nu * np.sqrt(np.asarray(self.gamma, dtype=np.float64))


def generate_channel(cfg: SystemConfig, rng: Rng) -> np.ndarray:
    """channel.cpp:7-16 (pure Python draws)."""
    cfg.validate()
    return random_matrix(cfg.K, cfg.M, rng)


def channel_for(cfg: SystemConfig, seed: int, stream: int) -> np.ndarray:
    """Fast path of test_pgd.cpp:30-34 through the C++ restatement."""
    cfg.validate()
    H = np.empty((cfg.M, cfg.K), dtype=np.complex128)
    rc = lib().ora_generate_channel(seed, stream, 1, cfg.K, cfg.M, _p(H))
    assert rc == ORA_OK
    return np.ascontiguousarray(H.T)


# --------------------------------------------------------------------------
# pgd.hpp / pgd.cpp
# --------------------------------------------------------------------------
@dataclass
class PgdParams:
    lambda_: float = 1.0 / 15.0
    eta: float = 0.0
    max_iters: int = 0
    residual_tol: float = 0.0
    trace_every: int = 0

    def validate(self):  # pgd.cpp:33-49
        if not (self.lambda_ >= 0.0):
            raise ValueError("PgdParams: lambda must be >= 0")
        if not (self.eta > 0.0):
            raise ValueError("PgdParams: eta must be > 0")
        if self.max_iters < 0:
            raise ValueError("PgdParams: max_iters must be >= 0")
        if not (self.residual_tol >= 0.0):
            raise ValueError("PgdParams: residual_tol must be >= 0")
        if self.trace_every < 0:
            raise ValueError("PgdParams: trace_every must be >= 0")


def mp_bound(num_users: int, num_antennas: int) -> float:
    out = C.c_double()
    if lib().ora_mp_bound(num_users, num_antennas, C.byref(out)) != ORA_OK:
        raise ValueError("mp_bound: dimensions must be positive")
    return out.value


def _check_shapes(H, cfg):
    cfg.validate()
    if H.shape != (cfg.K, cfg.M):
        raise ValueError("channel shape does not match SystemConfig")


def grad_f(W, H, cfg) -> np.ndarray:
    if W.shape != H.shape:
        raise ValueError("grad_f: precoder/channel shape mismatch")
    _check_shapes(H, cfg)
    K, M = H.shape
    c = cfg.constraint_diag()
    out = np.empty((M, K), dtype=np.complex128)
    lib().ora_grad_f(_p(to_storage(W)), _p(to_storage(H)), _p(c), K, M, _p(out))
    return from_storage(out, K, M)


def prox_l21(V, t: float) -> np.ndarray:
    if not (t >= 0.0):
        raise ValueError("prox_l21: threshold must be >= 0")
    K, M = V.shape
    out = np.empty((M, K), dtype=np.complex128)
    lib().ora_prox_l21(_p(to_storage(V)), K, M, float(t), _p(out))
    return from_storage(out, K, M)


def pgd_step(W, H, cfg, lambda_: float, eta: float) -> np.ndarray:
    if not (lambda_ >= 0.0) or not (eta > 0.0):
        raise ValueError("pgd_step: need lambda >= 0 and eta > 0")
    _check_shapes(H, cfg)
    K, M = H.shape
    out = np.empty((M, K), dtype=np.complex128)
    lib().ora_pgd_step(_p(to_storage(W)), _p(to_storage(H)), _p(cfg.constraint_diag()), K, M,
                       float(lambda_), float(eta), _p(out))
    return from_storage(out, K, M)


@dataclass
class LipschitzBound:
    exact: float = 0.0
    mp: float = 0.0


def lipschitz_bound(H, fixed_steps: int = 0) -> LipschitzBound:
    """pgd.cpp:120-169; fixed_steps > 0 is the BASELINE fixed-step rule."""
    K, M = H.shape
    if K < 1 or M < 1:
        raise ValueError("lipschitz_bound: empty channel")
    out = C.c_double()
    rc = lib().ora_lipschitz(_p(to_storage(H)), K, M, fixed_steps, C.byref(out))
    if rc == ORA_ECONVERGENCE:
        raise ConvergenceError("lipschitz_bound: power iteration did not reach tolerance")
    return LipschitzBound(out.value, mp_bound(K, M))


def power_v0(M: int) -> np.ndarray:
    v = np.empty(M, dtype=np.complex128)
    lib().ora_power_v0(M, _p(v))
    return v


def l21_norm(W) -> float:
    K, M = W.shape
    return lib().ora_l21_norm(_p(to_storage(W)), K, M)


def tx_power(W) -> float:
    return float(np.sum(np.abs(W) ** 2))


def consumed_power(W, alpha: float) -> float:
    if not (alpha > 0.0):
        raise ValueError("consumed_power: alpha must be > 0")
    return alpha * l21_norm(W)


def count_active_columns(W) -> int:
    K, M = W.shape
    return lib().ora_active_columns(_p(to_storage(W)), K, M)


def constraint_residual(H, W, cfg) -> float:
    K, M = H.shape
    return lib().ora_constraint_residual(_p(to_storage(H)), _p(to_storage(W)),
                                         _p(cfg.constraint_diag()), K, M)


def lagrangian_value(W, H, cfg, lambda_: float) -> float:
    K, M = H.shape
    return lib().ora_lagrangian(_p(to_storage(W)), _p(to_storage(H)), _p(cfg.constraint_diag()),
                                K, M, float(lambda_))


def zf_precoder(H, cfg) -> np.ndarray:
    _check_shapes(H, cfg)
    K, M = H.shape
    out = np.empty((M, K), dtype=np.complex128)
    rc = lib().ora_zf_precoder(_p(to_storage(H)), _p(cfg.constraint_diag()), K, M, _p(out))
    if rc == ORA_ESINGULAR:
        raise SingularChannelError("zf_precoder: channel Gram matrix is singular")
    return from_storage(out, K, M)


@dataclass
class MetricsReport:  # metrics.hpp:44-51
    tx_power: float
    cons_power: float
    sinr: np.ndarray
    sum_rate: float
    pcg: float
    residual: float


def compute_metrics(H, W, cfg) -> MetricsReport:
    """metrics.cpp:79-91 with the ZF reference computed here (zf.cpp:9-30)."""
    K, M = H.shape
    out = np.empty(6 + K)
    lib().ora_metrics(_p(to_storage(H)), _p(to_storage(W)), _p(cfg.constraint_diag()), cfg.sigma_nu, cfg.alpha,
                      K, M, _p(out))
    if out[5] == 0.0:
        raise SingularChannelError("zf_precoder: channel Gram matrix is singular")
    return MetricsReport(out[0], out[1], out[6:].copy(), out[2], out[3], out[4])


def sinr_per_user(H, W, cfg) -> np.ndarray:
    return compute_metrics(H, W, cfg).sinr


def sum_rate(sinr) -> float:
    return float(sum(math.log2(1.0 + s) for s in sinr))


def metrics_batch_f32(H, W, c, sigma_nu=1.0, alpha=1.0, threads=0):
    """[B, 6 + K]: tx, cons, sum_rate, pcg, residual, zf_ok, sinr[K]."""
    H = np.ascontiguousarray(H, dtype=np.complex64)
    W = np.ascontiguousarray(W, dtype=np.complex64)
    B, M, K = H.shape
    out = np.empty((B, 6 + K))
    c = np.ascontiguousarray(c, dtype=np.float64)
    rc = lib().ora_metrics_batch_f32(_p(H), _p(W), B, _p(c), float(sigma_nu), float(alpha), K, M, _p(out), threads)
    if rc != ORA_OK:
        raise ValueError("metrics batch failed")
    return out


def pcg(H, W, cfg) -> float:
    """metrics.cpp:56-69."""
    denom = l21_norm(W)
    if not (denom > 0.0):
        raise ValueError("pcg: precoder consumes zero power")
    return l21_norm(zf_precoder(H, cfg)) / denom


@dataclass
class PgdResult:
    precoder: np.ndarray
    iterations: int = 0


def solve_pgd(H, cfg, params: PgdParams, start=None) -> PgdResult:
    """pgd.cpp:178-268 (tracing is out of scope)."""
    _check_shapes(H, cfg)
    params.validate()
    K, M = H.shape
    if start is not None and start.shape != (K, M):
        raise ValueError("solve_pgd: W0 shape mismatch")
    out = np.empty((M, K), dtype=np.complex128)
    its, div = C.c_long(), C.c_long()
    w0 = None if start is None else to_storage(start)
    rc = lib().ora_solve_pgd(_p(to_storage(H)), _p(cfg.constraint_diag()), K, M, params.lambda_,
                             params.eta, params.max_iters, params.residual_tol, _p(w0), _p(out),
                             C.byref(its), C.byref(div))
    if rc == ORA_EDIVERGED:
        raise DivergenceError("solve_pgd: non-finite iterate", div.value)
    return PgdResult(from_storage(out, K, M), its.value)


def oracle_solve(H, cfg, lambda_: float) -> np.ndarray:
    """pgd.cpp:270-279."""
    p = PgdParams(lambda_, 1.0 / lipschitz_bound(H).exact, 100000, 1e-10, 0)
    return solve_pgd(H, cfg, p).precoder


# --------------------------------------------------------------------------
# unfolded.hpp / unfolded.cpp
# --------------------------------------------------------------------------
BOUND_SLACK = 1e-12  # unfolded.cpp:17


@dataclass
class LayerParams:
    lambda_i: float = 0.0
    eta_i: float = 0.0


@dataclass
class UnfoldedNetwork:
    num_users: int = 0
    num_antennas: int = 0
    mp_bound: float = 0.0
    layers: List[LayerParams] = field(default_factory=list)

    @staticmethod
    def pgd_init(num_users, num_antennas, num_layers, lambda_):  # unfolded.cpp:39-54
        if num_layers < 1:
            raise ValueError("pgd_init: need at least one layer")
        if not (lambda_ >= 0.0):
            raise ValueError("pgd_init: lambda must be >= 0")
        mp = mp_bound(num_users, num_antennas)
        net = UnfoldedNetwork(num_users, num_antennas, mp,
                              [LayerParams(lambda_, 1.0 / mp) for _ in range(num_layers)])
        net.validate()
        return net

    def validate(self):  # unfolded.cpp:56-69
        if self.num_users < 1 or self.num_antennas < self.num_users:
            raise ValueError("UnfoldedNetwork: bad dimensions")
        if not self.layers:
            raise ValueError("UnfoldedNetwork: no layers")
        expected = mp_bound(self.num_users, self.num_antennas)
        if not (abs(self.mp_bound - expected) <= 1e-9 * expected):
            raise ValueError("UnfoldedNetwork: mp_bound does not match (K, M)")


def check_projected(net: UnfoldedNetwork):  # unfolded.cpp:19-35
    hi = 1.0 / net.mp_bound
    lo = 0.5 * hi
    for i, layer in enumerate(net.layers):
        if not (layer.lambda_i >= 0.0) or not math.isfinite(layer.lambda_i):
            raise ValueError(f"UnfoldedNetwork: layer {i} lambda_i < 0")
        if not (layer.eta_i >= lo * (1.0 - BOUND_SLACK)) or not (layer.eta_i <= hi * (1.0 + BOUND_SLACK)):
            raise ValueError(f"UnfoldedNetwork: layer {i} eta_i outside [1/(2L), 1/L]")


def project_params(net: UnfoldedNetwork) -> UnfoldedNetwork:  # unfolded.cpp:71-81
    net.validate()
    hi = 1.0 / net.mp_bound
    lo = 0.5 * hi
    return UnfoldedNetwork(net.num_users, net.num_antennas, net.mp_bound,
                           [LayerParams(max(0.0, l.lambda_i), min(max(l.eta_i, lo), hi))
                            for l in net.layers])


@dataclass
class ForwardOptions:
    with_tape: bool = False
    with_iterates: bool = False


@dataclass
class LayerTape:
    input: np.ndarray
    step_image: np.ndarray
    column_norms: np.ndarray
    shrink_factors: np.ndarray


@dataclass
class ForwardResult:
    output: np.ndarray
    tape: List[LayerTape] = field(default_factory=list)
    iterates: List[np.ndarray] = field(default_factory=list)


def forward(net: UnfoldedNetwork, H, cfg: SystemConfig, start=None,
            options: ForwardOptions = ForwardOptions()) -> ForwardResult:
    """unfolded.cpp:83-150."""
    net.validate()
    check_projected(net)
    cfg.validate()
    if cfg.K != net.num_users or cfg.M != net.num_antennas or H.shape != (cfg.K, cfg.M):
        raise ValueError("forward: dimension mismatch")
    K, M = H.shape
    if start is not None and start.shape != (K, M):
        raise ValueError("forward: W0 shape mismatch")
    L = len(net.layers)
    lam = np.array([l.lambda_i for l in net.layers], dtype=np.float64)
    eta = np.array([l.eta_i for l in net.layers], dtype=np.float64)
    out = np.empty((M, K), dtype=np.complex128)
    div = C.c_long()
    its = np.empty((L + 1, M, K), dtype=np.complex128) if options.with_iterates else None
    tin = np.empty((L, M, K), dtype=np.complex128) if options.with_tape else None
    tv = np.empty((L, M, K), dtype=np.complex128) if options.with_tape else None
    tn = np.empty((L, M)) if options.with_tape else None
    ts = np.empty((L, M)) if options.with_tape else None
    w0 = None if start is None else to_storage(start)
    rc = lib().ora_forward(_p(to_storage(H)), _p(cfg.constraint_diag()), K, M, _p(lam), _p(eta), L,
                           _p(w0), _p(out), C.byref(div), _p(its), _p(tin), _p(tv), _p(tn), _p(ts))
    if rc == ORA_EDIVERGED:
        raise DivergenceError("forward: non-finite iterate at layer", div.value)
    res = ForwardResult(from_storage(out, K, M))
    if options.with_iterates:
        res.iterates = [from_storage(its[i], K, M) for i in range(L + 1)]
    if options.with_tape:
        res.tape = [LayerTape(from_storage(tin[i], K, M), from_storage(tv[i], K, M), tn[i].copy(),
                              ts[i].copy()) for i in range(L)]
    return res


def forward_infer(net, H, cfg) -> np.ndarray:
    return forward(net, H, cfg).output


@dataclass
class ParamGradients:
    d_lambda: np.ndarray
    d_eta: np.ndarray


def backward(tape: List[LayerTape], net: UnfoldedNetwork, H, cfg, dcost_dw) -> ParamGradients:
    """unfolded.cpp:158-239."""
    net.validate()
    cfg.validate()
    L = len(net.layers)
    K, M = H.shape
    if len(tape) != L:
        raise TrainingError("backward: tape depth does not match network")
    if dcost_dw.shape != (K, M) or H.shape != (cfg.K, cfg.M):
        raise TrainingError("backward: shape mismatch")
    lam = np.array([l.lambda_i for l in net.layers])
    eta = np.array([l.eta_i for l in net.layers])
    tin = np.stack([to_storage(t.input) for t in tape])
    tv = np.stack([to_storage(t.step_image) for t in tape])
    tn = np.stack([t.column_norms for t in tape]).astype(np.float64)
    ts = np.stack([t.shrink_factors for t in tape]).astype(np.float64)
    dl, de = np.empty(L), np.empty(L)
    rc = lib().ora_backward(_p(to_storage(H)), K, M, _p(lam), _p(eta), L, _p(tin), _p(tv), _p(tn), _p(ts),
                            _p(to_storage(dcost_dw)), _p(dl), _p(de))
    if rc != ORA_OK:
        raise TrainingError("backward: layer step size must be > 0")
    return ParamGradients(dl, de)


def unsupervised_loss(W, H, cfg, lambda_cost) -> float:  # training.cpp:76-81
    return lagrangian_value(W, H, cfg, lambda_cost)


def unsupervised_loss_grad(W, H, cfg, lambda_cost) -> np.ndarray:  # training.cpp:83-95
    g = 2.0 * grad_f(W, H, cfg)
    for m in range(W.shape[1]):
        n = np.linalg.norm(W[:, m])
        if n > 0.0:
            g[:, m] += (lambda_cost / n) * W[:, m]
    return g


def train_batch_f32(H, c, lam, eta, loss_kind=0, lambda_cost=1.0 / 15.0, labels=None, threads=0):
    """Per-sample loss and (d_lambda_i, d_eta_i) of train's inner loop
    (training.cpp:205-234) over complex64 channels [B][M][K]."""
    H = np.ascontiguousarray(H, dtype=np.complex64)
    B, M, K = H.shape
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    eta = np.ascontiguousarray(eta, dtype=np.float64)
    L = lam.size
    loss = np.empty(B)
    grads = np.empty((B, 2 * L))
    st = np.empty(B, dtype=np.int32)
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.complex64)
    rc = lib().ora_train_batch_f32(_p(H), B, _p(np.ascontiguousarray(c, dtype=np.float64)), K, M, _p(lam), _p(eta), L,
                                   loss_kind, float(lambda_cost), _p(lab), _p(loss), _p(grads), _p(st), threads)
    if rc != ORA_OK:
        raise ValueError("train batch failed")
    return loss, grads, st


# --------------------------------------------------------------------------
# Batched drivers (complex64 inputs [B][M][K], the GPU's layout)
# --------------------------------------------------------------------------
def default_thread_count() -> int:
    return lib().ora_default_thread_count()


def forward_batch_f32(H: np.ndarray, c: np.ndarray, lam: np.ndarray, eta: np.ndarray,
                      w0_mode: int = 0, W0: Optional[np.ndarray] = None, threads: int = 0,
                      want_W: bool = True):
    """H: complex64 [B][M][K]. Returns dict with W (complex128 [B][M][K]),
    diverged_at, l21, active, tie_margin."""
    H = np.ascontiguousarray(H, dtype=np.complex64)
    B, M, K = H.shape
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    eta = np.ascontiguousarray(eta, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    W = np.empty((B, M, K), dtype=np.complex128) if want_W else None
    div = np.empty(B, dtype=np.int32)
    l21 = np.empty(B)
    act = np.empty(B, dtype=np.int32)
    tie = np.empty(B)
    w0 = None if W0 is None else np.ascontiguousarray(W0, dtype=np.complex64)
    rc = lib().ora_forward_batch_f32(_p(H), B, _p(c), K, M, _p(lam), _p(eta), len(lam), w0_mode,
                                     _p(w0), _p(W), _p(div), _p(l21), _p(act), _p(tie), threads)
    if rc != ORA_OK:
        raise ValueError(f"ora_forward_batch_f32 failed: {rc}")
    return dict(W=W, diverged_at=div, l21=l21, active=act, tie_margin=tie)


def pgd_batch_f32(H: np.ndarray, c: np.ndarray, lambda_: float, eta: np.ndarray, max_iters: int,
                  residual_tol: float = 0.0, w0_mode: int = 1, W0=None, threads: int = 0,
                  want_W: bool = True):
    H = np.ascontiguousarray(H, dtype=np.complex64)
    B, M, K = H.shape
    eta = np.ascontiguousarray(eta, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    W = np.empty((B, M, K), dtype=np.complex128) if want_W else None
    div = np.empty(B, dtype=np.int32)
    its = np.empty(B, dtype=np.int64)
    l21 = np.empty(B)
    act = np.empty(B, dtype=np.int32)
    tie = np.empty(B)
    w0 = None if W0 is None else np.ascontiguousarray(W0, dtype=np.complex64)
    rc = lib().ora_pgd_batch_f32(_p(H), B, _p(c), K, M, float(lambda_), _p(eta), max_iters,
                                 residual_tol, w0_mode, _p(w0), _p(W), _p(div), _p(its), _p(l21),
                                 _p(act), _p(tie), threads)
    if rc != ORA_OK:
        raise ValueError(f"ora_pgd_batch_f32 failed: {rc}")
    return dict(W=W, diverged_at=div, iterations=its, l21=l21, active=act, tie_margin=tie)


def generate_channels_batch_f32(seed_h: int, seed_g: int, gain_range_db: float, first: int, B: int, K: int,
                                M: int, threads: int = 0) -> np.ndarray:
    """The BASELINE workloads' seeded channels as complex64
    [B][M][K]: channel.cpp:7-16 draws with log-uniform user gains."""
    H = np.empty((B, M, K), dtype=np.complex64)
    rc = lib().ora_generate_channels_batch_f32(seed_h, seed_g, float(gain_range_db), first, B, K, M, _p(H), threads)
    if rc != ORA_OK:
        raise ValueError("ora_generate_channels_batch_f32 failed")
    return H


def layer_params(seed_p: int, L: int, K: int, M: int):
    """Raw seeded (lambda_l, mu_l) of SURVEY §8d (before project_params)."""
    lam, eta = np.empty(L), np.empty(L)
    if lib().ora_layer_params(seed_p, L, K, M, _p(lam), _p(eta)) != ORA_OK:
        raise ValueError("ora_layer_params failed")
    return lam, eta


def power_iteration_batch_f32(H: np.ndarray, steps: int = 30, threads: int = 0):
    H = np.ascontiguousarray(H, dtype=np.complex64)
    B, M, K = H.shape
    L = np.empty(B)
    st = np.empty(B, dtype=np.int32)
    rc = lib().ora_power_iteration_batch_f32(_p(H), B, K, M, steps, _p(L), _p(st), threads)
    if rc != ORA_OK:
        raise ValueError(f"ora_power_iteration_batch_f32 failed: {rc}")
    return L, st


def lagrangian_batch(H: np.ndarray, W: np.ndarray, c: np.ndarray, lambda_: float, threads: int = 0):
    H = np.ascontiguousarray(H, dtype=np.complex64)
    B, M, K = H.shape
    c = np.ascontiguousarray(c, dtype=np.float64)
    out = np.empty(B)
    if W.dtype == np.complex64:
        W = np.ascontiguousarray(W)
        rc = lib().ora_lagrangian_batch_f32(_p(H), _p(W), B, _p(c), K, M, float(lambda_), _p(out), threads)
    else:
        W = np.ascontiguousarray(W, dtype=np.complex128)
        rc = lib().ora_lagrangian_batch_f64(_p(H), _p(W), B, _p(c), K, M, float(lambda_), _p(out), threads)
    if rc != ORA_OK:
        raise ValueError("lagrangian batch failed")
    return out


# --------------------------------------------------------------------------
# training.cpp:140-308 — the train loop over the FP64 per-sample restatement
# (ora_train_batch_f32) with the reference's shuffle stream, ordered batch
# means, Adam (training.cpp:116-138) and projection (training.cpp:33-38).
# --------------------------------------------------------------------------
SHUFFLE_STREAM = 0x7D5A1E0B33C4F216  # training.cpp:20


def shuffle(items: list, rng: Rng) -> None:
    """rng.hpp:43-50 Fisher-Yates."""
    for i in range(len(items), 1, -1):
        j = rng.index_below(i)
        items[i - 1], items[j] = items[j], items[i - 1]


def adam_update(state: dict, grads, params, lr: float) -> None:
    for i, g in enumerate(grads):
        if not math.isfinite(g):
            raise ValueError(f"adam_update: non-finite gradient for parameter {i}")
    state["step"] += 1
    b1, b2, eps = 0.9, 0.999, 1e-8
    bias1 = 1.0 - b1 ** state["step"]
    bias2 = 1.0 - b2 ** state["step"]
    m, v = state["m"], state["v"]
    for i, g in enumerate(grads):
        m[i] = b1 * m[i] + (1.0 - b1) * g
        v[i] = b2 * v[i] + (1.0 - b2) * g * g
        params[i] -= lr * (m[i] / bias1) / (math.sqrt(v[i] / bias2) + eps)


def train_loop_f32(train_H, val_H, c, lam0, eta0, *, loss_kind=0, lambda_cost=1.0 / 15.0, batch_size=64,
                   learning_rate=1e-3, max_epochs=200, patience=10, seed=0, train_labels=None, val_labels=None,
                   sigma_nu=1.0, alpha=1.0, threads=0):
    """Complex64 datasets [N][M][K]; returns dict(epochs=[(epoch, train_loss,
    val_loss, val_pcg, val_sum_rate)], best_epoch, stopping_epoch, params)."""
    N, M, K = train_H.shape
    hi = 1.0 / mp_bound(K, M)
    lo = 0.5 * hi
    params = []
    for lmb, et in zip(lam0, eta0):  # project_params, packed (training.hpp:50-51)
        params += [max(0.0, lmb), min(max(et, lo), hi)]
    state = dict(step=0, m=[0.0] * len(params), v=[0.0] * len(params))
    rng = Rng.stream(seed, SHUFFLE_STREAM)
    order = list(range(N))
    epochs, best_val, best_epoch, best_params, since, stop = [], math.inf, -1, None, 0, -1
    for epoch in range(max_epochs):
        shuffle(order, rng)
        loss_sum = 0.0
        for start in range(0, N, batch_size):
            idx = order[start:start + batch_size]
            lam, eta = np.array(params[0::2]), np.array(params[1::2])
            lab = None if train_labels is None else train_labels[idx]
            loss, grads, _ = train_batch_f32(train_H[idx], c, lam, eta, loss_kind, lambda_cost, lab, threads)
            n = len(idx)
            batch_loss = 0.0
            mean = [0.0] * len(params)
            for b in range(n):  # ordered reduction (training.cpp:236-246)
                batch_loss += loss[b]
                for p in range(len(params)):
                    mean[p] += grads[b, p]
            batch_loss /= n
            mean = [g / n for g in mean]
            if not math.isfinite(batch_loss):
                raise ValueError(f"train: non-finite loss at epoch {epoch}")
            loss_sum += batch_loss * n
            adam_update(state, mean, params, learning_rate)
            for i in range(0, len(params), 2):
                params[i] = max(0.0, params[i])
                params[i + 1] = min(max(params[i + 1], lo), hi)
        lam, eta = np.array(params[0::2]), np.array(params[1::2])
        W = forward_batch_f32(val_H, c, lam, eta, w0_mode=1, threads=threads)["W"]
        rows = metrics_batch_f32(val_H, W, c, sigma_nu, alpha, threads)
        if loss_kind == 1:
            vl = np.sum(np.abs(W - val_labels) ** 2, axis=(1, 2))
        else:
            vl = lambda_cost * rows[:, 1] / alpha + rows[:, 4] ** 2
        rec = (epoch, loss_sum / N, float(np.mean(vl)), float(np.mean(rows[:, 3])), float(np.mean(rows[:, 2])))
        epochs.append(rec)
        stop = epoch
        if rec[2] < best_val:
            best_val, best_epoch, best_params, since = rec[2], epoch, list(params), 0
        else:
            since += 1
        if since >= patience:
            break
    return dict(epochs=epochs, best_epoch=best_epoch, stopping_epoch=stop, params=best_params)
