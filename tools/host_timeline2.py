"""Cross-call chunk timeline of streamed host calls (development aid):
UFPGD_OPT_HOST_TIMELINE = 2 prints each call's chunks at its wait, on the
first call's clock."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2304_12745_b200 as U
w = U.CONFIGS[2]
H = torch.from_numpy(U.make_inputs(w)).pin_memory().numpy()
Ws = [torch.empty(H.shape, dtype=torch.complex64).pin_memory().numpy() for _ in range(3)]
lam, eta = w.layer_params()
for _ in range(2): U.unfolded_forward_host(H, lam, eta, w.c, out=Ws[0])
U.set_option("host_timeline", 2)
prev = None
for k in range(int(os.environ.get("NCALLS", "4"))):
    cur = U.unfolded_forward_host_async(H, lam, eta, w.c, out=Ws[k % 3])
    if prev is not None: prev.wait()
    prev = cur
prev.wait()
