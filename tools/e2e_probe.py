"""End-to-end host-buffer throughput of config 2 (development aid; bench.py's e2e leg)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_12745_b200 as U

if os.environ.get("UFPGD_HOST_CHUNK_MB"):  # tuning sweep input of this probe (tools/e2e_ab.sh)
    U.set_option("host_chunk_bytes", int(os.environ["UFPGD_HOST_CHUNK_MB"]) << 20)
if os.environ.get("UFPGD_E2E_PIPE"):  # 1: the depth-first streams pipeline (A/B)
    U.set_option("host_pipe", int(os.environ["UFPGD_E2E_PIPE"]))
w = U.CONFIGS[2]
H = torch.from_numpy(U.make_inputs(w)).pin_memory()
W = torch.empty_like(H).pin_memory()
lam, eta = w.layer_params()
Hn, Wn = H.numpy(), W.numpy()
for _ in range(2):
    U.unfolded_forward_host(Hn, lam, eta, w.c, w0_mode=w.w0_mode, out=Wn)
best = 0.0
for _ in range(3):
    t0 = time.perf_counter()
    for _ in range(10):
        U.unfolded_forward_host(Hn, lam, eta, w.c, w0_mode=w.w0_mode, out=Wn)
    best = max(best, 10 * w.B / (time.perf_counter() - t0))
print(f"e2e chunk={os.environ.get('UFPGD_HOST_CHUNK_MB', 'default')} MB: {best / 1e6:.2f} M precoders/s", flush=True)
