"""Generates tests/golden/fixtures.npz — committed golden vectors for the
parity tests (run from the repo root: python tests/golden/make_golden.py).

* The 2x4 scripted fixtures of test_pgd.cpp:247-308 and
  test_unfolded.cpp:134-180, evaluated here by the same scalar loops the
  reference tests use (pure Python, no library code): these are independent
  known answers.
* Seeded BASELINE-shaped cases (config 1 and config 2 layer parameters, a
  config-3 PGD run) evaluated by the FP64 oracle: regression pins of the
  oracle itself, which is pinned to the reference by tests/test_oracle_*.py.
* Random-source known answers: std::mt19937_64 and Rng::stream draws.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2304_12745_b200 as U  # noqa: E402
from _support import fixture_2x4, scripted_layer  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    out = {}
    cfg, h = fixture_2x4()
    target = [0.8 * np.sqrt(2.0), 0.8 * np.sqrt(0.5)]
    out["fx_H"] = h
    out["fx_c"] = cfg.constraint_diag()
    one, _, _ = scripted_layer(h.conj(), h, target, 1.5, 0.05)
    out["fx_step_lambda_eta"] = np.array([1.5, 0.05])
    out["fx_step_W"] = one
    layers = [(0.9, 0.05), (1.5, 0.07), (0.3, 0.08)]
    w = h.conj()
    for lam, eta in layers:
        w, _, _ = scripted_layer(w, h, target, lam, eta)
    out["fx_layers"] = np.array(layers)
    out["fx_forward_W"] = w
    out["mp_bound_8_64"] = np.array([117.25483399593904])

    g = O.MT19937_64(5489)
    out["mt19937_64_first4"] = np.array([g() for _ in range(4)], dtype=np.uint64)
    r = O.Rng.stream(1002, 0)
    out["rng_stream_1002_0_cn"] = np.array([r.complex_gaussian() for _ in range(8)])
    out["power_v0_64"] = O.power_v0(64)

    for cfg_id, n in [(1, 8), (2, 8)]:
        wl = U.CONFIGS[cfg_id]
        H = U.make_inputs(wl, 0, n)
        lam, eta = wl.layer_params()
        ora = O.forward_batch_f32(H, wl.c, lam, eta, w0_mode=wl.w0_mode, threads=1)
        out[f"cfg{cfg_id}_H"] = H
        out[f"cfg{cfg_id}_lambda"] = lam
        out[f"cfg{cfg_id}_eta"] = eta
        out[f"cfg{cfg_id}_W"] = ora["W"]
        out[f"cfg{cfg_id}_l21"] = ora["l21"]

    wl = U.CONFIGS[3]
    H = U.make_inputs(wl, 0, 4)
    L30, _ = O.power_iteration_batch_f32(H, wl.power_steps, threads=1)
    ora = O.pgd_batch_f32(H, wl.c, wl.lambda_pgd, 1.0 / L30, 200, w0_mode=wl.w0_mode, threads=1)
    out["cfg3_H"] = H
    out["cfg3_L30"] = L30
    out["cfg3_iters"] = np.array([200])
    out["cfg3_W"] = ora["W"]
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "fixtures.npz"), **out)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
