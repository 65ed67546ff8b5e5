"""FP64 oracle (the reference's CPU path restated) timed on the host cores for
every BASELINE config, on bounded seeded samples (development aid; bench.py
times config 2 itself). Prints one line per config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2304_12745_b200 as U
from oracle import oracle as O

threads = O.default_thread_count()
for cfg, n, secs in ((1, 1024, 5.0), (2, 4096, 5.0), (3, 64, 10.0), (4, 256, 10.0), (5, 2048, 10.0)):
    w = U.CONFIGS[cfg]
    H = U.make_inputs(w, 0, n)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < secs:
        if w.kind == "pgd":
            L = O.power_iteration_batch_f32(H, w.power_steps, threads=threads)[0]
            O.pgd_batch_f32(H, w.c, w.lambda_pgd, 1.0 / np.asarray(L), w.L, threads=threads, want_W=False)
        else:
            lam, eta = w.layer_params()
            O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode, threads=threads, want_W=False)
        done += n
    rate = done / (time.perf_counter() - t0)
    print(f"cfg{cfg}: {rate:,.0f} precoders/s on {threads} threads ({1e6 / rate * threads:.1f} core-us per realization)",
          flush=True)
