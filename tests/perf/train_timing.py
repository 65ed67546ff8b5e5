"""Training-loop timing (development aid): ufpgd::train on the device via
build/train_dump vs the oracle's restated loop on the host cores, same data."""
import math, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2304_12745_b200 as U
from oracle import oracle as O
import _ufpd

K, M, L, NT, NV, EP = 8, 64, 20, 2048, 256, 3
Ht = U.generate_channels(600, 0, 0.0, 0, NT, K, M)
Hv = U.generate_channels(601, 0, 0.0, 0, NV, K, M)
_ufpd.write("/tmp/tt_tr.ufpd", np.transpose(Ht, (0, 2, 1)).astype(np.complex128))
_ufpd.write("/tmp/tt_va.ufpd", np.transpose(Hv, (0, 2, 1)).astype(np.complex128))
t0 = time.perf_counter()
out = subprocess.run(["build/train_dump", "/tmp/tt_tr.ufpd", "/tmp/tt_va.ufpd", str(L), repr(1 / 15), "0", repr(1 / 15),
                      "64", "1e-3", str(EP), "10", "3"], capture_output=True, text=True,
                     env=dict(os.environ, UFPGD_TRAIN_WARMUP="1"))
td = time.perf_counter() - t0
assert out.returncode == 0, out.stderr
import json
tt = json.loads(out.stdout)["train_seconds"]
t0 = time.perf_counter()
O.train_loop_f32(Ht, Hv, np.full(K, math.sqrt(10.0)), [1 / 15] * L, [1 / O.mp_bound(K, M)] * L, batch_size=64,
                 learning_rate=1e-3, max_epochs=EP, patience=10, seed=3)
to = time.perf_counter() - t0
print(f"train (8,64) L=20, {NT} train / {NV} val, batch 64, {EP} epochs: device train() {tt:.3f} s "
      f"(process incl. CUDA init + file read {td:.2f} s), oracle loop {to:.2f} s on {O.default_thread_count()} threads")
