for v in base ch2 base ch2; do echo "== $v"; UFPGD_LIB=tools/ablib/$v/libufpgd_gpu.so python - <<'PY'
import math, time, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_12745_b200 as U
K, M = 8, 64
c = np.full(K, math.sqrt(10.0))
H = U.generate_channels_device(33, 0, 0.0, 0, 8192, K, M, dtype=torch.complex128)
U.oracle_solve(H[:8].contiguous(), c, 1/15, max_iters=1000); torch.cuda.synchronize()
t0 = time.perf_counter(); out = U.oracle_solve(H, c, 1/15, max_iters=20000); torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"8192 x 2e4 iters: {dt:.3f} s  {8192*2e4/dt/1e6:.1f} M realization-iterations/s")
PY
done
