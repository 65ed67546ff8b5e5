"""Copy/compute pipeline shapes over PCIe (development aid): 256 MiB each way
in chunks over `ns` streams, with a per-chunk device sleep standing in for the
kernel; issue orders: depth-first (H2D, kernel, D2H per chunk) or skewed
(H2D + kernel of chunk k, then D2H of chunk k - 1)."""
import time, torch
n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); w = torch.empty(n, dtype=torch.uint8).pin_memory()
for ns in (4,):
  for cmb in (16, 32):
    c = cmb << 20
    st = [torch.cuda.Stream() for _ in range(ns)]
    dh = [torch.empty(c, dtype=torch.uint8, device="cuda") for _ in range(ns)]
    dw = [torch.empty(c, dtype=torch.uint8, device="cuda") for _ in range(ns)]
    N = n // c
    def run(compute, order):
      if order == "depth":
        for k in range(N):
          i = k % ns
          with torch.cuda.stream(st[i]):
            dh[i].copy_(h[k*c:(k+1)*c], non_blocking=True)
            if compute: torch.cuda._sleep(compute)
            w[k*c:(k+1)*c].copy_(dw[i], non_blocking=True)
      else:
        for k in range(N + 1):
          if k < N:
            i = k % ns
            with torch.cuda.stream(st[i]):
              dh[i].copy_(h[k*c:(k+1)*c], non_blocking=True)
              if compute: torch.cuda._sleep(compute)
          if k >= 1:
            j = (k - 1) % ns
            with torch.cuda.stream(st[j]):
              w[(k-1)*c:k*c].copy_(dw[j], non_blocking=True)
      torch.cuda.synchronize()
    for order in ("depth", "skew"):
      for comp in (0, 200000):
        run(comp, order); t0 = time.perf_counter(); run(comp, order); t = time.perf_counter() - t0
        print(f"ns={ns} chunk={cmb}MB {order} sleep={comp}: {t*1e3:.2f} ms  {2*n/t/1e9:.1f} GB/s total", flush=True)
