"""Per-call completion periods of streamed host calls (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2304_12745_b200 as U
w = U.CONFIGS[2]
H = torch.from_numpy(U.make_inputs(w)).pin_memory().numpy()
NB = int(os.environ.get("NBUF", "3"))
Ws = [torch.empty(H.shape, dtype=torch.complex64).pin_memory().numpy() for _ in range(NB)]
lam, eta = w.layer_params()
for k in range(3): U.unfolded_forward_host(H, lam, eta, w.c, out=Ws[k % NB])
for rep in range(3):
    ts = []; prev = None
    t0 = time.perf_counter()
    for k in range(16):
        cur = U.unfolded_forward_host_async(H, lam, eta, w.c, out=Ws[k % NB])
        te = time.perf_counter()
        if prev is not None:
            prev.wait(); ts.append((time.perf_counter() - t0) * 1e3)
        prev = cur
        if k == 0: enq = (te - t0) * 1e3
    prev.wait(); ts.append((time.perf_counter() - t0) * 1e3)
    per = [round(b - a, 2) for a, b in zip(ts, ts[1:])]
    print(f"rep {rep}: enqueue {enq:.2f} ms, first done {ts[0]:.2f}, periods {per}, total {ts[-1]:.2f}", flush=True)
