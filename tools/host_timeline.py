import os, sys
sys.path.insert(0, ".")
import torch, paper_2304_12745_b200 as U
w = U.CONFIGS[2]
H = torch.from_numpy(U.make_inputs(w)).pin_memory(); W = torch.empty_like(H).pin_memory()
lam, eta = w.layer_params()
for _ in range(2): U.unfolded_forward_host(H.numpy(), lam, eta, w.c, out=W.numpy())
U.set_option("host_timeline", 1)
U.unfolded_forward_host(H.numpy(), lam, eta, w.c, out=W.numpy())
