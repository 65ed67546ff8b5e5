"""One unfolded_forward launch of a config (for ncu A/B captures; development aid).
  python tools/one_launch.py CFG [B]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_12745_b200 as U

cfg = int(sys.argv[1])
w = U.CONFIGS[cfg]
B = int(sys.argv[2]) if len(sys.argv) > 2 else w.B
H = U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, B, w.K, w.M)
lam, eta = w.layer_params()
W = torch.empty_like(H)
for _ in range(2):
    U.unfolded_forward(H, lam, eta, w.c, out=W)
torch.cuda.synchronize()
