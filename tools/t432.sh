for v in tm4 tm2 tm8 tm16; do echo "== $v"; UFPGD_LIB=tools/ablib/$v/libufpgd_gpu.so python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_12745_b200 as U
K, M = 4, 32
lam, eta = U.project_params(*U.layer_params(3, 20, K, M), K, M)
c = np.full(K, np.sqrt(10.0))
for B in (1024, 65536):
    H = U.generate_channels_device(7, 0, 0.0, 0, B, K, M); W = torch.empty_like(H)
    run = lambda: U.unfolded_forward(H, lam, eta, c, out=W)
    run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): run()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50): g.replay()
    e.record(); torch.cuda.synchronize()
    print(f"B={B}: {s.elapsed_time(e)/50*1e3:.1f} us")
PY
done
