"""B200-native batched PA-aware precoder solver (arXiv 2304.12745 hot path).

Python bindings over the C ABI in ``include/ufpgd_gpu.h`` (built into
``paper_2304_12745_b200/lib/libufpgd_gpu.so`` for sm_100a). Torch provides
device memory and streams; every computation runs in the hand-written CUDA
kernels of ``csrc/*.cu``. There is no CPU fallback: importing works
without a GPU, but every compute call raises if the library or the device is
missing.

Batches use the reference's storage: complex64 tensors of shape [B, M, K]
(Eigen col-major K x M per realization, column m = antenna m;
/root/reference/proj/core/include/ufpgd/types.hpp:14-20).
"""
from __future__ import annotations

from .capi import (  # noqa: F401
    ConvergenceError,
    DataFormatError,
    DivergenceError,
    UfpgdError,
    W0_CONJ_H,
    W0_GIVEN,
    W0_ZERO,
    abi_version,
    get_option,
    options,
    set_option,
    fp32_peak,
    init_multi_gpu,
    shutdown_multi_gpu,
    unfolded_forward_sharded,
    unfolded_forward_sharded_device,
    generate_channels,
    generate_channels_device,
    layer_params,
    layers_general,
    lipschitz_exact,
    metrics,
    oracle_solve,
    summarize_metrics,
    lib,
    lib_path,
    pgd_fixed,
    pgd_fixed_host,
    power_iteration,
    power_v0,
    unfolded_forward,
    unfolded_forward_host,
    unfolded_forward_host_async,
    unfolded_grad,
    unfolded_backward64,
    ufpd_header,
    ufpd_load,
    ufpd_store,
)
from .workloads import CONFIGS, Workload, make_inputs, mp_bound, project_params  # noqa: F401
