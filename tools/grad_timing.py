import sys, time, torch
sys.path.insert(0, ".")
import paper_2304_12745_b200 as U
w = U.CONFIGS[2]
lam, eta = w.layer_params()
for B in (64, 256, 1024, 4096):
    H = torch.from_numpy(U.make_inputs(w, 0, B)).cuda()
    for _ in range(3): U.unfolded_grad(H, lam, eta, w.c)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): U.unfolded_grad(H, lam, eta, w.c)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"grad B={B}: {ms:.3f} ms  ({B/ms*1e3/1e3:.1f} k samples/s)")
