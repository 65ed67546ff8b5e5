"""ctypes bindings of the C ABI (include/ufpgd_gpu.h).

Every entry point here maps one-to-one onto an ``extern "C"`` function of
``libufpgd_gpu.so``; status codes become the reference's exception types
(errors.hpp:8-39): ``ValueError`` for ``std::invalid_argument``,
``DivergenceError(index)`` and ``ConvergenceError``.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# UFPGD_LIB overrides the library path (A/B builds of the same ABI in tools/).
_LIB = os.environ.get("UFPGD_LIB") or os.path.join(_HERE, "lib", "libufpgd_gpu.so")

OK, EINVAL_SHAPE, EINVAL_PARAM, EDIVERGED, ECONVERGENCE, ECUDA, ENCCL, ENOTSUP, EDATAFORMAT = (
    0, -1, -2, -3, -4, -5, -6, -7, -8)
W0_ZERO, W0_CONJ_H, W0_GIVEN = 0, 1, 2


class UfpgdError(RuntimeError):
    """A CUDA / NCCL / unsupported-shape failure of the product library."""


class DivergenceError(RuntimeError):
    """errors.hpp:18-25 — non-finite iterate; ``index`` is the 0-based layer
    (forward) or 1-based iteration (solve_pgd) of the first failure."""

    def __init__(self, what: str, index: int, per_realization=None):
        super().__init__(what)
        self.index = index
        self.diverged_at = per_realization


class ConvergenceError(RuntimeError):
    pass


class DataFormatError(RuntimeError):
    """errors.hpp:33-37 — malformed or truncated dataset file."""


_lib = None


def lib_path() -> str:
    return _LIB


def lib():
    """Loads the CUDA library; raises (never falls back) when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} is missing: run `make` (or __graft_entry__.build()) first; "
                              "there is no CPU fallback for the ufpgd hot path")
        L = C.CDLL(_LIB)
        i, d, i64, u64, P = C.c_int, C.c_double, C.c_int64, C.c_uint64, C.c_void_p
        sigs = {
            "ufpgd_gpu_abi_version": (i, []),
            "ufpgd_gpu_set_option": (i, [i, i64]),
            "ufpgd_gpu_get_option": (i64, [i]),
            "ufpgd_gpu_last_error": (C.c_char_p, []),
            "ufpgd_gpu_device_count": (i, [P]),
            "ufpgd_gpu_unfolded_forward": (i, [P, i64, i, i, P, P, i, P, i, P, P, P, P, P, P, d, i, P]),
            "ufpgd_gpu_power_iteration": (i, [P, i64, i, i, P, i, P, i, P]),
            "ufpgd_gpu_pgd_fixed": (i, [P, i64, i, i, P, i, d, i64, P, i, P, P, P, P, P, P, P, d, i, P]),
            "ufpgd_gpu_solve_pgd_batch": (i, [P, i64, i, i, P, i, d, i64, d, P, i, P, P, P, P, P, P, P, P, d, i, P]),
            "ufpgd_gpu_layers_general": (i, [P, i64, i, i, P, P, i, P, i, P, i, d, i, P, P, P, P, P, P, P, i, P]),
            "ufpgd_gpu_unfolded_forward_host": (i, [P, i64, i, i, P, P, i, P, i, P, P, P, P, d, i]),
            "ufpgd_gpu_unfolded_forward_host_async": (i, [P, i64, i, i, P, P, i, P, i, P, P, P, P, d, i, P]),
            "ufpgd_gpu_host_wait": (i, [i64]),
            "ufpgd_gpu_pgd_fixed_host": (i, [P, i64, i, i, i, d, i64, P, i, P, P, P, P, P, d, i]),
            "ufpgd_gpu_fp32_peak": (i, [i, P, P]),
            "ufpgd_dataset_last_error": (C.c_char_p, []),
            "ufpgd_ufpd_read_header": (i, [C.c_char_p, P, P, P, P, P]),
            "ufpgd_gpu_ufpd_load": (i, [C.c_char_p, i64, i64, i, P, i]),
            "ufpgd_gpu_ufpd_store": (i, [C.c_char_p, i, i, i64, u64, P, P, i]),
            "ufpgd_gpu_convert_f64_rowmajor": (i, [P, i64, i, i, P, i, i, P]),
            "ufpgd_gpu_metrics": (i, [P, P, i64, i, i, P, d, d, P, P, i, P]),
            "ufpgd_gpu_layers_general64": (i, [P, i64, i, i, P, P, i, P, i, P, i, d, i, P, P, P, P, P, P, P, i, P]),
            "ufpgd_gpu_solve_pgd64": (i, [P, i64, i, i, P, d, P, i64, d, P, P, P, P, i, P]),
            "ufpgd_gpu_oracle_solve": (i, [P, i64, i, i, P, d, i64, d, P, P, P, P, i, P]),
            "ufpgd_gpu_unfolded_grad": (i, [P, i64, i, i, P, P, i, P, i, i, d, P, P, P, P, i, P]),
            "ufpgd_gpu_unfolded_backward64": (i, [P, i64, i, i, P, P, i, P, i, P, P, P, i, P]),
            "ufpgd_gpu_init": (i, [i]),
            "ufpgd_gpu_shutdown": (i, []),
            "ufpgd_gpu_unfolded_forward_sharded": (i, [P, i64, i, i, P, P, i, P, i, P, P, P, P, d]),
            "ufpgd_gpu_unfolded_forward_sharded_device": (i, [P, P, i, i, P, P, i, P, i, P, P, P, P, d, P]),
            "ufpgd_gpu_lipschitz_exact": (i, [P, i64, i, i, P, P, i, P]),
            "ufpgd_power_v0_f64": (i, [i, P]),
            "ufpgd_generate_channels": (i, [u64, u64, d, i64, i64, i, i, P, i]),
            "ufpgd_gpu_generate_channels": (i, [u64, u64, d, i64, i64, i, i, P, i, i, P]),
            "ufpgd_power_v0": (i, [i, P]),
            "ufpgd_layer_params": (i, [u64, i, i, i, P, P]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def abi_version() -> int:
    return lib().ufpgd_gpu_abi_version()


# ufpgd_gpu_set_option ids (include/ufpgd_gpu.h): explicit, process-wide
# tuning / A-B switches; the library never reads them from the environment.
OPTIONS = {"tensor_cores": 0, "fused_warps": 1, "fp64_team": 2, "zero_pad": 3, "pad_sub_bytes": 4,
           "host_pipe": 5, "host_chunk_bytes": 6, "host_timeline": 7}


def set_option(name: str, value: int) -> None:
    if name not in OPTIONS:
        raise ValueError(f"unknown option {name!r}")
    _check(lib().ufpgd_gpu_set_option(OPTIONS[name], int(value)))


def get_option(name: str) -> int:
    if name not in OPTIONS:
        raise ValueError(f"unknown option {name!r}")
    return int(lib().ufpgd_gpu_get_option(OPTIONS[name]))


class options:
    """Context manager: ``with options(tensor_cores=0): ...`` sets library
    options for the block and restores the previous values."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_option(k, v)
        return False


def _check(rc: int, diverged=None, index_base: int = 0):
    if rc == OK:
        return
    msg = lib().ufpgd_gpu_last_error().decode()
    if rc in (EINVAL_SHAPE, EINVAL_PARAM):
        raise ValueError(msg)
    if rc == EDIVERGED:
        idx = -1
        if diverged is not None:
            d = np.asarray(diverged)
            bad = d[d >= 0]
            idx = int(bad.min()) if bad.size else -1
        raise DivergenceError(msg, idx, diverged)
    if rc == ECONVERGENCE:
        raise ConvergenceError(msg)
    raise UfpgdError(f"ufpgd status {rc}: {msg}")


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


def _stream_ptr(stream, device=None) -> Optional[int]:
    """The launch stream: ``stream`` or the current stream OF THE TENSOR'S
    DEVICE (the C ABI launches on that device; another device's stream handle
    would be rejected as an invalid resource)."""
    import torch

    if stream is not None:
        if device is not None and stream.device != device:
            raise ValueError(f"stream is on {stream.device}, the batch on {device}")
        return stream.cuda_stream
    return torch.cuda.current_stream(device).cuda_stream


def _check_batch(H):
    import torch

    if not (isinstance(H, torch.Tensor) and H.is_cuda and H.dtype == torch.complex64 and H.dim() == 3
            and H.is_contiguous()):
        raise ValueError("H must be a contiguous CUDA complex64 tensor [B, M, K]")
    B, M, K = H.shape
    return B, K, M


def _check_like(t, H, name: str):
    """A device operand the kernels index like H (W0, out): same shape,
    dtype, device and contiguity, else the reference's shape error
    (unfolded.cpp:96-99, pgd.cpp:184-187) instead of an out-of-bounds access."""
    import torch

    if t is None:
        return
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.device == H.device and t.dtype == H.dtype
            and tuple(t.shape) == tuple(H.shape) and t.is_contiguous()):
        raise ValueError(f"{name} shape mismatch: need a contiguous {H.dtype} tensor {tuple(H.shape)} on {H.device}")


def _check_host_like(a, H, name: str):
    """Host operand (W0, out) of the host-buffer entry points: C-contiguous
    complex64 numpy array of H's shape."""
    if a is None:
        return
    if not (isinstance(a, np.ndarray) and a.dtype == np.complex64 and a.shape == H.shape and a.flags.c_contiguous
            and (name != "out" or a.flags.writeable)):
        raise ValueError(f"{name} shape mismatch: need a C-contiguous complex64 array {H.shape}")


def _check_w0(w0_mode: int, W0, H, host: bool = False):
    if w0_mode not in (W0_ZERO, W0_CONJ_H, W0_GIVEN):
        raise ValueError(f"w0_mode must be 0, 1 or 2 (got {w0_mode})")
    if w0_mode == W0_GIVEN and W0 is None:
        raise ValueError("w0_mode = W0_GIVEN needs W0")
    (_check_host_like if host else _check_like)(W0, H, "W0")


def unfolded_forward(H, lambda_, eta, c, *, w0_mode: int = W0_ZERO, W0=None, alpha: float = 1.0,
                     want_stats: bool = True, want_per_realization: bool = False, out=None,
                     stream=None):
    """Batched ufpgd::forward (unfolded.cpp:83-156) on device tensors.

    Returns dict(W=[B,M,K] complex64, diverged_at=int32[B], l21, active,
    stats=float64[3]) with the optional entries None when not requested.
    Asynchronous on ``stream``; divergence is reported in ``diverged_at`` /
    ``stats[2]`` rather than raised (the caller decides, as with the reference's
    per-index slots)."""
    import torch

    B, K, M = _check_batch(H)
    lam, et, cc = _f64(lambda_), _f64(eta), _f64(c)
    if lam.size != et.size:
        raise ValueError("lambda and eta must have one entry per layer")
    _check_w0(w0_mode, W0, H)
    _check_like(out, H, "out")
    dev = H.device
    W = out if out is not None else torch.empty_like(H)
    div = torch.empty(B, dtype=torch.int32, device=dev)
    l21 = torch.empty(B, dtype=torch.float32, device=dev) if want_per_realization else None
    act = torch.empty(B, dtype=torch.int32, device=dev) if want_per_realization else None
    stats = torch.empty(3, dtype=torch.float64, device=dev) if want_stats else None
    rc = lib().ufpgd_gpu_unfolded_forward(
        _ptr(H), B, K, M, _ptr(lam), _ptr(et), lam.size, _ptr(cc), w0_mode, _ptr(W0), _ptr(W), _ptr(div),
        _ptr(l21), _ptr(act), _ptr(stats), float(alpha), dev.index or 0, _stream_ptr(stream, dev))
    _check(rc)
    return dict(W=W, diverged_at=div, l21=l21, active=act, stats=stats)


def power_iteration(H, steps: int = 30, v0=None, stream=None):
    """Batched fixed-step lipschitz_bound (pgd.cpp:120-169, BASELINE 30-step rule)."""
    import torch

    B, K, M = _check_batch(H)
    Lout = torch.empty(B, dtype=torch.float32, device=H.device)
    v = None if v0 is None else np.ascontiguousarray(v0, dtype=np.complex64)
    if v is not None and v.shape != (M,):
        raise ValueError(f"v0 must have M = {M} entries")
    rc = lib().ufpgd_gpu_power_iteration(_ptr(H), B, K, M, _ptr(v), steps, _ptr(Lout), H.device.index or 0,
                                         _stream_ptr(stream, H.device))
    _check(rc)
    return Lout


def pgd_fixed(H, lambda_: float, iters: int, c, *, eta=None, power_steps: int = 30,
              w0_mode: int = W0_CONJ_H, W0=None, alpha: float = 1.0, want_per_realization=False,
              residual_tol: float = 0.0, stream=None):
    """Batched ufpgd::solve_pgd at a fixed step (pgd.cpp:178-268, trace off):
    ``iters`` iterations, or fewer per realization with ``residual_tol`` > 0
    (relative iterate change, pgd.cpp:246-260; ``iterations`` then holds the
    counts). ``eta`` (device float32 [B]) or the in-kernel 1/L."""
    import torch

    B, K, M = _check_batch(H)
    cc = _f64(c)
    _check_w0(w0_mode, W0, H)
    if eta is not None and not (isinstance(eta, torch.Tensor) and eta.is_cuda and eta.device == H.device
                                and eta.dtype == torch.float32 and tuple(eta.shape) == (B,) and eta.is_contiguous()):
        raise ValueError(f"eta must be a contiguous CUDA float32 tensor [{B}] on {H.device}")
    dev = H.device
    W = torch.empty_like(H)
    div = torch.empty(B, dtype=torch.int32, device=dev)
    eta_out = torch.empty(B, dtype=torch.float32, device=dev)
    l21 = torch.empty(B, dtype=torch.float32, device=dev) if want_per_realization else None
    act = torch.empty(B, dtype=torch.int32, device=dev) if want_per_realization else None
    stats = torch.empty(3, dtype=torch.float64, device=dev)
    its = torch.empty(B, dtype=torch.int64, device=dev) if (want_per_realization or residual_tol > 0) else None
    rc = lib().ufpgd_gpu_solve_pgd_batch(_ptr(H), B, K, M, _ptr(eta), power_steps, float(lambda_), int(iters),
                                         float(residual_tol), _ptr(cc), w0_mode, _ptr(W0), _ptr(W), _ptr(div),
                                         _ptr(its), _ptr(l21), _ptr(act), _ptr(eta_out), _ptr(stats), float(alpha),
                                         dev.index or 0, _stream_ptr(stream, dev))
    _check(rc)
    return dict(W=W, diverged_at=div, eta=eta_out, l21=l21, active=act, stats=stats, iterations=its)


def layers_general(H, eta, thr, c, *, w0_mode: int = W0_CONJ_H, W0=None, mode: int = 0,
                   residual_tol: float = 0.0, index_base: int = 0, iterates: bool = False,
                   tape: bool = False, stream=None):
    """General-shape layer sweep with raw (eta, thr) per layer and optional
    tapes (unfolded.hpp:40-62); mode 1 returns grad_f(W0) (pgd.cpp:68-83)."""
    import torch

    B, K, M = _check_batch(H)
    et, th, cc = _f64(eta), _f64(thr), _f64(c)
    _check_w0(w0_mode, W0, H)
    L = 1 if mode == 1 else et.size
    dev = H.device
    W = torch.empty_like(H)
    div = torch.empty(B, dtype=torch.int32, device=dev)
    its = torch.empty(B, dtype=torch.int64, device=dev)
    itr = torch.empty((L + 1, B, M, K), dtype=torch.complex64, device=dev) if iterates else None
    tv = torch.empty((L, B, M, K), dtype=torch.complex64, device=dev) if tape else None
    tn = torch.empty((L, B, M), dtype=torch.float32, device=dev) if tape else None
    ts = torch.empty((L, B, M), dtype=torch.float32, device=dev) if tape else None
    rc = lib().ufpgd_gpu_layers_general(
        _ptr(H), B, K, M, _ptr(et), _ptr(th), L, _ptr(cc), w0_mode, _ptr(W0), mode, float(residual_tol),
        index_base, _ptr(W), _ptr(div), _ptr(its), _ptr(itr), _ptr(tv), _ptr(tn), _ptr(ts),
        dev.index or 0, _stream_ptr(stream, dev))
    _check(rc)
    return dict(W=W, diverged_at=div, iterations=its, iterates=itr, tape_v=tv, tape_norms=tn,
                tape_shrink=ts)


def unfolded_forward_host(H: np.ndarray, lambda_, eta, c, *, w0_mode: int = W0_ZERO, W0=None,
                          alpha: float = 1.0, out: Optional[np.ndarray] = None, device: int = 0,
                          raise_on_divergence: bool = True):
    """End-to-end host-buffer forward (pipelined H2D / kernel / D2H)."""
    H = np.asarray(H)
    if H.dtype != np.complex64 or H.ndim != 3 or not H.flags.c_contiguous:
        raise ValueError("H must be a C-contiguous complex64 array [B, M, K]")
    B, M, K = H.shape
    lam, et, cc = _f64(lambda_), _f64(eta), _f64(c)
    _check_w0(w0_mode, W0, H, host=True)
    _check_host_like(out, H, "out")
    W = out if out is not None else np.empty_like(H)
    div = np.empty(B, dtype=np.int32)
    stats = np.zeros(3)
    rc = lib().ufpgd_gpu_unfolded_forward_host(_ptr(H), B, K, M, _ptr(lam), _ptr(et), lam.size, _ptr(cc),
                                               w0_mode, _ptr(W0), _ptr(W), _ptr(div), _ptr(stats),
                                               float(alpha), device)
    if rc == EDIVERGED and not raise_on_divergence:
        rc = OK
    _check(rc, div)
    return dict(W=W, diverged_at=div, stats=stats)


class HostCall:
    """An enqueued host-buffer call (unfolded_forward_host_async): ``wait()``
    blocks until its W, diverged_at and stats are in the host buffers and
    raises DivergenceError like the synchronous call (unless told not to).
    Keeps its buffers alive until then."""

    def __init__(self, ticket, W, div, stats, keep):
        self.ticket, self.W, self.diverged_at, self.stats, self._keep = ticket, W, div, stats, keep
        self._done = False

    def wait(self, raise_on_divergence: bool = True):
        if not self._done:
            rc = lib().ufpgd_gpu_host_wait(self.ticket)
            self._done = True
            if rc == EDIVERGED and not raise_on_divergence:
                rc = OK
            _check(rc, self.diverged_at)
        return dict(W=self.W, diverged_at=self.diverged_at, stats=self.stats)


def unfolded_forward_host_async(H: np.ndarray, lambda_, eta, c, *, w0_mode: int = W0_ZERO, W0=None,
                                alpha: float = 1.0, out: Optional[np.ndarray] = None, device: int = 0) -> HostCall:
    """Enqueue-only host-buffer forward: back-to-back calls overlap one batch's
    copy-out with the next batch's copy-in (H, W0 and out should be pinned)."""
    H = np.asarray(H)
    if H.dtype != np.complex64 or H.ndim != 3 or not H.flags.c_contiguous:
        raise ValueError("H must be a C-contiguous complex64 array [B, M, K]")
    B, M, K = H.shape
    lam, et, cc = _f64(lambda_), _f64(eta), _f64(c)
    _check_w0(w0_mode, W0, H, host=True)
    _check_host_like(out, H, "out")
    W = out if out is not None else np.empty_like(H)
    div = np.empty(B, dtype=np.int32)
    stats = np.zeros(3)
    ticket = C.c_int64(-1)
    rc = lib().ufpgd_gpu_unfolded_forward_host_async(_ptr(H), B, K, M, _ptr(lam), _ptr(et), lam.size, _ptr(cc),
                                                     w0_mode, _ptr(W0), _ptr(W), _ptr(div), _ptr(stats),
                                                     float(alpha), device, C.byref(ticket))
    _check(rc)
    return HostCall(ticket.value, W, div, stats, (H, W0))


def pgd_fixed_host(H: np.ndarray, lambda_: float, iters: int, c, *, power_steps: int = 30,
                   w0_mode: int = W0_CONJ_H, W0=None, alpha: float = 1.0, device: int = 0,
                   raise_on_divergence: bool = True):
    H = np.asarray(H)
    if H.dtype != np.complex64 or H.ndim != 3 or not H.flags.c_contiguous:
        raise ValueError("H must be a C-contiguous complex64 array [B, M, K]")
    B, M, K = H.shape
    cc = _f64(c)
    _check_w0(w0_mode, W0, H, host=True)
    W = np.empty_like(H)
    div = np.empty(B, dtype=np.int32)
    eta = np.empty(B, dtype=np.float32)
    stats = np.zeros(3)
    rc = lib().ufpgd_gpu_pgd_fixed_host(_ptr(H), B, K, M, power_steps, float(lambda_), int(iters), _ptr(cc),
                                        w0_mode, _ptr(W0), _ptr(W), _ptr(div), _ptr(eta), _ptr(stats),
                                        float(alpha), device)
    if rc == EDIVERGED and not raise_on_divergence:
        rc = OK
    _check(rc, div, 1)
    return dict(W=W, diverged_at=div, eta=eta, stats=stats)


def lipschitz_exact(H, stream=None):
    """Converged FP64 power iteration (pgd.cpp:120-169) for a complex128 CUDA
    tensor [B, M, K]; returns (L float64[B], status int32[B])."""
    import torch

    if not (isinstance(H, torch.Tensor) and H.is_cuda and H.dtype == torch.complex128 and H.dim() == 3
            and H.is_contiguous()):
        raise ValueError("H must be a contiguous CUDA complex128 tensor [B, M, K]")
    B, M, K = H.shape
    Lout = torch.empty(B, dtype=torch.float64, device=H.device)
    st = torch.empty(B, dtype=torch.int32, device=H.device)
    _check(lib().ufpgd_gpu_lipschitz_exact(_ptr(H), B, K, M, _ptr(Lout), _ptr(st), H.device.index or 0,
                                           _stream_ptr(stream, H.device)))
    return Lout, st


def metrics(H, W, c, *, sigma_nu: float = 1.0, alpha: float = 1.0, want_zf: bool = False, stream=None):
    """Batched compute_metrics + ZF reference (metrics.cpp:79-91, zf.cpp:9-30)
    on device tensors [B, M, K]. Returns dict(out=float64 [B, 6 + K] with
    columns tx_power, cons_power, sum_rate, pcg, residual, zf_ok, sinr..., zf)."""
    import torch

    B, K, M = _check_batch(H)
    _check_like(W, H, "W")
    cc = _f64(c)
    out = torch.empty((B, 6 + K), dtype=torch.float64, device=H.device)
    zf = torch.empty_like(H) if want_zf else None
    _check(lib().ufpgd_gpu_metrics(_ptr(H), _ptr(W), B, K, M, _ptr(cc), float(sigma_nu), float(alpha), _ptr(out),
                                   _ptr(zf), H.device.index or 0, _stream_ptr(stream, H.device)))
    return dict(out=out, zf=zf)


def unfolded_grad(H, lambda_, eta, c, *, w0_mode: int = W0_CONJ_H, loss_kind: int = 0,
                  lambda_cost: float = 1.0 / 15.0, labels=None, stream=None):
    """Per-sample loss and parameter gradients of train's inner loop
    (training.cpp:205-234) for device channels [B, M, K]; returns dict(loss
    [B], grads [B, 2L] in pack order, mean [1 + 2L])."""
    import torch

    B, K, M = _check_batch(H)
    lam, et, cc = _f64(lambda_), _f64(eta), _f64(c)
    _check_like(labels, H, "labels")
    L = lam.size
    loss = torch.empty(B, dtype=torch.float64, device=H.device)
    grads = torch.empty((B, 2 * L), dtype=torch.float64, device=H.device)
    mean = torch.empty(1 + 2 * L, dtype=torch.float64, device=H.device)
    _check(lib().ufpgd_gpu_unfolded_grad(_ptr(H), B, K, M, _ptr(lam), _ptr(et), L, _ptr(cc), w0_mode, loss_kind,
                                         float(lambda_cost), _ptr(labels), _ptr(loss), _ptr(grads), _ptr(mean),
                                         H.device.index or 0, _stream_ptr(stream, H.device)))
    return dict(loss=loss, grads=grads, mean=mean)


def summarize_metrics(out):
    """evaluate's reduction (training.cpp:361-399): means and standard errors
    of tx_power, cons_power, sinr, sum_rate, pcg, residual over realizations."""
    o = np.asarray(out, dtype=np.float64)
    n = len(o)
    cols = {"tx_power": o[:, 0], "cons_power": o[:, 1], "sum_rate": o[:, 2], "pcg": o[:, 3], "residual": o[:, 4]}
    mean = {k: float(v.mean()) for k, v in cols.items()}
    mean["sinr"] = o[:, 6:].mean(axis=0)
    se = {}
    if n > 1:
        scale = 1.0 / ((n - 1) * n)
        se = {k: float(np.sqrt(((v - mean[k]) ** 2).sum() * scale)) for k, v in cols.items()}
        se["sinr"] = np.sqrt(((o[:, 6:] - mean["sinr"]) ** 2).sum(axis=0) * scale)
    return {"num_channels": n, "mean": mean, "std_error": se}


def _check_data(rc):
    if rc == EDATAFORMAT:
        raise DataFormatError(lib().ufpgd_dataset_last_error().decode())
    if rc != OK:
        msg = lib().ufpgd_dataset_last_error().decode() or lib().ufpgd_gpu_last_error().decode()
        if rc in (EINVAL_SHAPE, EINVAL_PARAM):
            raise ValueError(msg)
        raise UfpgdError(f"ufpgd status {rc}: {msg}")


def ufpd_header(path: str) -> dict:
    """Header of a UFPD dataset file (dataset.hpp:23-33); host only."""
    K, M, N, seed, lab = C.c_int(), C.c_int(), C.c_int64(), C.c_uint64(), C.c_int()
    _check_data(lib().ufpgd_ufpd_read_header(path.encode(), C.byref(K), C.byref(M), C.byref(N), C.byref(seed),
                                             C.byref(lab)))
    return dict(K=K.value, M=M.value, N=N.value, seed=seed.value, has_labels=bool(lab.value))


def ufpd_load(path: str, first: int = 0, count=None, labels: bool = False, device: int = 0):
    """Samples of a UFPD file as a CUDA complex64 batch [count, M, K]."""
    import torch

    h = ufpd_header(path)
    n = h["N"] - first if count is None else count
    out = torch.empty((n, h["M"], h["K"]), dtype=torch.complex64, device=f"cuda:{device}")
    _check_data(lib().ufpgd_gpu_ufpd_load(path.encode(), first, n, 1 if labels else 0, _ptr(out), device))
    return out


def ufpd_store(path: str, channels, labels=None, seed: int = 0, device: int = 0):
    """write_dataset from CUDA complex64 batches [N, M, K] (labels optional)."""
    N, M, K = channels.shape
    if labels is not None and tuple(labels.shape) != tuple(channels.shape):
        raise ValueError("write_dataset: label shape mismatch")
    _check_data(lib().ufpgd_gpu_ufpd_store(path.encode(), K, M, N, seed, _ptr(channels), _ptr(labels), device))


def oracle_solve(H, c, lambda_: float, *, max_iters: int = 100000, residual_tol: float = 1e-10, stream=None):
    """oracle_solve at scale (pgd.cpp:270-279) in FP64 for a complex128 CUDA
    batch [B, M, K]: returns dict(W complex128, eta, iterations, status)."""
    import torch

    if not (isinstance(H, torch.Tensor) and H.is_cuda and H.dtype == torch.complex128 and H.dim() == 3
            and H.is_contiguous()):
        raise ValueError("H must be a contiguous CUDA complex128 tensor [B, M, K]")
    B, M, K = H.shape
    W = torch.empty_like(H)
    eta = torch.empty(B, dtype=torch.float64, device=H.device)
    its = torch.empty(B, dtype=torch.int64, device=H.device)
    st = torch.empty(B, dtype=torch.int32, device=H.device)
    _check(lib().ufpgd_gpu_oracle_solve(_ptr(H), B, K, M, _ptr(_f64(c)), float(lambda_), int(max_iters),
                                        float(residual_tol), _ptr(W), _ptr(eta), _ptr(its), _ptr(st),
                                        H.device.index or 0, _stream_ptr(stream, H.device)))
    return dict(W=W, eta=eta, iterations=its, status=st)


def fp32_peak(device: int = 0):
    """Measured FP32 FMA peak (TFLOP/s) with the fused kernel's FFMA2 form and
    the SM clock (GHz) observed during the probe."""
    t, g = C.c_double(), C.c_double()
    _check(lib().ufpgd_gpu_fp32_peak(device, C.byref(t), C.byref(g)))
    return t.value, g.value


def init_multi_gpu(ngpus: int):
    _check(lib().ufpgd_gpu_init(ngpus))


def shutdown_multi_gpu():
    _check(lib().ufpgd_gpu_shutdown())


def unfolded_forward_sharded(H: np.ndarray, lambda_, eta, c, *, w0_mode: int = W0_ZERO, W0=None,
                             alpha: float = 1.0, raise_on_divergence: bool = True):
    """Single-process multi-GPU forward over the devices given to
    init_multi_gpu, from host buffers: contiguous shards, one NCCL all-reduce
    of the statistics."""
    H = np.asarray(H)
    if H.dtype != np.complex64 or H.ndim != 3 or not H.flags.c_contiguous:
        raise ValueError("H must be a C-contiguous complex64 array [B, M, K]")
    B, M, K = H.shape
    lam, et, cc = _f64(lambda_), _f64(eta), _f64(c)
    _check_w0(w0_mode, W0, H, host=True)
    W = np.empty_like(H)
    div = np.empty(B, dtype=np.int32)
    stats = np.zeros(3)
    rc = lib().ufpgd_gpu_unfolded_forward_sharded(_ptr(H), B, K, M, _ptr(lam), _ptr(et), lam.size, _ptr(cc),
                                                  w0_mode, _ptr(W0), _ptr(W), _ptr(div), _ptr(stats), float(alpha))
    if rc == EDIVERGED and not raise_on_divergence:
        rc = OK
    _check(rc, div)
    return dict(W=W, diverged_at=div, stats=stats)


def unfolded_forward_sharded_device(shards, lambda_, eta, c, *, w0_mode: int = W0_ZERO, W0=None,
                                    alpha: float = 1.0, streams=None):
    """Single-process multi-GPU forward over device-resident shards: shards[g]
    is a CUDA complex64 tensor [B_g, M, K] on device g (g < the count given to
    init_multi_gpu); W0 likewise for W0_GIVEN. Asynchronous on streams[g] (the
    current stream of each device by default). Returns dict of per-device
    lists W, diverged_at, stats — every stats[g] holds the global sums after
    the in-place NCCL all-reduce."""
    import torch

    G = len(shards)
    if G == 0:
        raise ValueError("need one shard per device")
    K = M = None
    for g, t in enumerate(shards):
        B, K_, M_ = _check_batch(t)
        if t.device.index != g:
            raise ValueError(f"shard {g} must live on cuda:{g}")
        if K is None:
            K, M = K_, M_
        elif (K_, M_) != (K, M):
            raise ValueError("all shards need the same (K, M)")
    if W0 is not None:
        if len(W0) != G:
            raise ValueError("W0 needs one tensor per shard")
        for g in range(G):
            _check_like(W0[g], shards[g], "W0")
    if w0_mode == W0_GIVEN and W0 is None:
        raise ValueError("w0_mode = W0_GIVEN needs W0")
    lam, et, cc = _f64(lambda_), _f64(eta), _f64(c)
    W = [torch.empty_like(t) for t in shards]
    div = [torch.empty(t.shape[0], dtype=torch.int32, device=t.device) for t in shards]
    stats = [torch.empty(3, dtype=torch.float64, device=t.device) for t in shards]
    arr = lambda xs: (C.c_void_p * G)(*[_ptr(x) for x in xs])  # noqa: E731
    Bs = (C.c_int64 * G)(*[t.shape[0] for t in shards])
    st = (C.c_void_p * G)(*[_stream_ptr(None if streams is None else streams[g], shards[g].device)
                            for g in range(G)])
    rc = lib().ufpgd_gpu_unfolded_forward_sharded_device(
        arr(shards), Bs, K, M, _ptr(lam), _ptr(et), lam.size, _ptr(cc), w0_mode,
        None if W0 is None else arr(W0), arr(W), arr(div), arr(stats), float(alpha), st)
    _check(rc)
    return dict(W=W, diverged_at=div, stats=stats)


def generate_channels(seed_h: int, seed_g: int, gain_range_db: float, first_index: int, B: int, K: int,
                      M: int, threads: int = 0, out: Optional[np.ndarray] = None) -> np.ndarray:
    """Seeded complex64 channels [B, M, K] (host; harness input, not timed)."""
    H = out if out is not None else np.empty((B, M, K), dtype=np.complex64)
    rc = lib().ufpgd_generate_channels(seed_h, seed_g, float(gain_range_db), first_index, B, K, M, _ptr(H),
                                       threads)
    _check(rc)
    return H


def generate_channels_device(seed_h: int, seed_g: int, gain_range_db: float, first_index: int, B: int, K: int,
                             M: int, *, dtype=None, device: int = 0, out=None, stream=None):
    """The same seeded draw generated on the device:
    a CUDA tensor [B, M, K], complex64 (default) or complex128. Async on
    ``stream``; bit-identical integer streams, FP64 entries within a few ulp of
    the host draw (CUDA log/sincos vs glibc)."""
    import torch

    dt = dtype if dtype is not None else torch.complex64
    if dt not in (torch.complex64, torch.complex128):
        raise ValueError("dtype must be complex64 or complex128")
    H = out if out is not None else torch.empty((B, M, K), dtype=dt, device=f"cuda:{device}")
    if out is not None and not (H.is_cuda and H.dtype == dt and tuple(H.shape) == (B, M, K) and H.is_contiguous()):
        raise ValueError("out must be a contiguous CUDA tensor [B, M, K] of the requested dtype")
    rc = lib().ufpgd_gpu_generate_channels(seed_h, seed_g, float(gain_range_db), first_index, B, K, M, _ptr(H),
                                           int(dt == torch.complex128), H.device.index or 0, _stream_ptr(stream, H.device))
    _check(rc)
    return H


def unfolded_backward64(H, lambda_, eta, c, dcost_dw, *, w0_mode: int = W0_CONJ_H, W0=None, stream=None):
    """backward (unfolded.cpp:158-239) in FP64 for complex128 CUDA batches
    [B, M, K]: the forward from W0 is re-run on the device with its tape and
    swept back from dcost_dw. Returns grads [B, 2L] in pack order."""
    import torch

    for t in (H, dcost_dw) + ((W0,) if W0 is not None else ()):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.complex128 and t.dim() == 3
                and t.is_contiguous()):
            raise ValueError("H, dcost_dw (and W0) must be contiguous CUDA complex128 tensors [B, M, K]")
    B, M, K = H.shape
    lam, et, cc = _f64(lambda_), _f64(eta), _f64(c)
    grads = torch.empty((B, 2 * lam.size), dtype=torch.float64, device=H.device)
    _check(lib().ufpgd_gpu_unfolded_backward64(_ptr(H), B, K, M, _ptr(lam), _ptr(et), lam.size, _ptr(cc), w0_mode,
                                               _ptr(W0), _ptr(dcost_dw), _ptr(grads), H.device.index or 0,
                                               _stream_ptr(stream, H.device)))
    return grads


def power_v0(M: int) -> np.ndarray:
    v = np.empty(M, dtype=np.complex64)
    _check(lib().ufpgd_power_v0(M, _ptr(v)))
    return v


def layer_params(seed_p: int, L: int, K: int, M: int):
    lam = np.empty(L)
    eta = np.empty(L)
    _check(lib().ufpgd_layer_params(seed_p, L, K, M, _ptr(lam), _ptr(eta)))
    return lam, eta
