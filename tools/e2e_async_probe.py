"""Streamed vs synchronous host-buffer calls (development aid): total time of
N back-to-back config-2 batches; the slope is the steady-state cost per batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_12745_b200 as U

w = U.CONFIGS[2]
H = torch.from_numpy(U.make_inputs(w)).pin_memory().numpy()
Ws = [torch.empty(H.shape, dtype=torch.complex64).pin_memory().numpy() for _ in range(3)]
lam, eta = w.layer_params()


def run(n, streamed):
    t0 = time.perf_counter()
    prev = None
    for k in range(n):
        if streamed:
            cur = U.unfolded_forward_host_async(H, lam, eta, w.c, out=Ws[k % 3])
            if prev is not None:
                prev.wait()
            prev = cur
        else:
            U.unfolded_forward_host(H, lam, eta, w.c, out=Ws[0])
    if prev is not None:
        prev.wait()
    return (time.perf_counter() - t0) * 1e3


for streamed in (False, True):
    run(4, streamed)
    res = {n: min(run(n, streamed) for _ in range(3)) for n in (1, 2, 4, 8, 16)}
    slope = (res[16] - res[4]) / 12
    print(f"{'streamed' if streamed else 'sync    '}: " + "  ".join(f"N={n}: {t:6.2f} ms" for n, t in res.items())
          + f"  -> {slope:.3f} ms per batch ({w.B / slope / 1e3:.2f} M/s steady state)", flush=True)
