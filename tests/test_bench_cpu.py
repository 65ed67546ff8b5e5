"""bench.py contract checks that run without a GPU: the reference arm
(`--impl reference`, the FP64 oracle port on the host cores) prints one JSON
line with the fields the driver reads, and the cost model / geometry helpers
are consistent."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # the whole per-GPU batch per step, described with the GPU arm's config keys
    assert d["config"]["per_gpu_batch"] == d["config"]["global_batch"] == 65536
    assert d["config"]["layers_eta_clamped_by_projection"] == 7


def test_reference_arm_loads_no_product_library():
    """Inputs and layer parameters come from oracle/ (the restatements of
    channel.cpp:7-16 / rng.cpp:19-40), so only oracle libraries are mapped."""
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0'];"
            "import bench; bench.main();"
            "maps = open('/proc/self/maps').read();"
            "print('PRODUCT_SO', 'libufpgd_gpu' in maps, 'ORACLE_SO', 'libufpgd_oracle' in maps)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "PRODUCT_SO False ORACLE_SO True" in r.stdout


def test_oracle_inputs_equal_product_inputs():
    """The reference arm's oracle-generated batch and projected parameters are
    the GPU arm's, bit for bit."""
    sys.path.insert(0, ROOT)
    import numpy as np

    import bench
    import paper_2304_12745_b200 as U
    from oracle import oracle as O

    for cfg in (2, 5):
        w = U.CONFIGS[cfg]
        a = U.make_inputs(w, 1234, 64)
        b = O.generate_channels_batch_f32(w.seed_h, w.seed_g, w.gain_db, 1234, 64, w.K, w.M)
        assert np.array_equal(a, b)
        lam, eta, clamped = bench.projected_params_oracle(w)
        lam2, eta2 = w.layer_params()
        assert np.array_equal(lam, lam2) and np.array_equal(eta, eta2)
        assert clamped == bench.clamped_layers(w)


def test_cost_model_counts_performed_contractions():
    sys.path.insert(0, ROOT)
    import paper_2304_12745_b200 as U

    w = U.CONFIGS[2]
    K, M, L = w.K, w.M, w.L
    assert w.flops_per_realization() == (2 * L - 2) * 8 * K * K * M + 10 * K * M * L
    assert w.flops_per_realization(exact_w0=False) == 2 * L * 8 * K * K * M + 10 * K * M * L
    assert w.bytes_per_realization() == 16 * K * M


def test_tensor_core_flop_model():
    """Tensor-core flops of the tcgen05 kernel (csrc/mma.cu) per realization:
    stage 1 M=4K, N=4K, K=M (skipped at a W0 = 0 layer 0), stage 2 per
    128-antenna tile M=128, N=4K+2K, K=2K; ~3x the FP32-equivalent work (the
    3-term f16 split) plus the stage-1 lo*lo block."""
    sys.path.insert(0, ROOT)
    import paper_2304_12745_b200 as U

    for cfg in (4, 5):
        w = U.CONFIGS[cfg]
        K, M, L = w.K, w.M, w.L
        s1 = 2 * (4 * K) * (4 * K) * M
        s2 = (M // 128) * 2 * 128 * (6 * K) * (2 * K)
        assert w.tensor_flops_per_realization() == (L - 1) * s1 + L * s2
        assert 2.5 < w.tensor_flops_per_realization() / w.flops_per_realization() < 4.5
    # config 2: (8,64) realization pairs in the (16,128) frame, each with its own
    # stage-1 chain (M 64, N 32, K 64) and stage-2 K-step (M 128, N 32 + 16, K 16)
    w2 = U.CONFIGS[2]
    s1 = 2 * 64 * 32 * 64
    s2 = 2 * 128 * 48 * 16
    assert w2.tensor_flops_per_realization() == (w2.L - 1) * s1 + w2.L * s2
    # the 3-term split's ~3x, times ~2 for the frame rows each MMA still carries
    assert 5 < w2.tensor_flops_per_realization() / w2.flops_per_realization() < 8
    for cfg in (1, 3):
        assert U.CONFIGS[cfg].tensor_flops_per_realization() is None


def test_measured_peaks_fallback():
    sys.path.insert(0, ROOT)
    import bench

    p = bench.measured_peaks()
    assert p["hbm_gbs"] > 1000 and p["bf16_tflops"] > 500
    assert p["source"] in ("MEASURED_PEAKS.json", "fallback")
