"""Copy engines vs kernels (development aid): 256 MiB each way in 16 MiB chunks.
indep: all H2D on one stream, all D2H on another, no dependencies (optionally
with sleep kernels running on a third stream); split: H2D -> sleep -> D2H per
chunk chained by events over separate copy-in / kernel / copy-out streams."""
import time, torch
n, c = 256 << 20, 16 << 20
N = n // c
h = torch.empty(n, dtype=torch.uint8).pin_memory(); w = torch.empty(n, dtype=torch.uint8).pin_memory()
dh = [torch.empty(c, dtype=torch.uint8, device="cuda") for _ in range(N)]
dw = [torch.empty(c, dtype=torch.uint8, device="cuda") for _ in range(N)]
S = [torch.cuda.Stream() for _ in range(6)]

def indep(sleep, nin=1, nout=1):
    for k in range(N):
        with torch.cuda.stream(S[k % nin]): dh[k].copy_(h[k*c:(k+1)*c], non_blocking=True)
        with torch.cuda.stream(S[2 + k % nout]): w[k*c:(k+1)*c].copy_(dw[k], non_blocking=True)
        if sleep:
            with torch.cuda.stream(S[4]): torch.cuda._sleep(sleep)

def split(sleep, nin=2, nout=2):
    for k in range(N):
        si, sk, so = S[k % nin], S[4 + (k & 1)], S[2 + k % nout]
        with torch.cuda.stream(si): dh[k].copy_(h[k*c:(k+1)*c], non_blocking=True)
        sk.wait_stream(si)
        with torch.cuda.stream(sk):
            if sleep: torch.cuda._sleep(sleep)
        so.wait_stream(sk)
        with torch.cuda.stream(so): w[k*c:(k+1)*c].copy_(dw[k], non_blocking=True)

def timeit(f):
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best

for name, f in [("indep copy-only 1+1", lambda: indep(0)), ("indep copy-only 2+2", lambda: indep(0, 2, 2)),
                ("indep + sleeps", lambda: indep(200000)), ("split no-sleep 2+2", lambda: split(0)),
                ("split sleep 2+2", lambda: split(200000)), ("split sleep 1+1", lambda: split(200000, 1, 1)),
                ("split sleep=50k 2+2", lambda: split(50000))]:
    t = timeit(f)
    print(f"{name:24s} {t*1e3:6.2f} ms  {2*n/t/1e9:5.1f} GB/s", flush=True)

# per-chunk timelines: the split pipeline with sleeps, and the independent copies
def timeline(kind):
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(N)]
    t0 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    S[0].record_event(t0)
    for x in S[1:]: x.wait_event(t0)
    for k in range(N):
        si, sk, so = (S[0], S[4 + (k & 1)], S[2]) if kind != "split2" else (S[k % 2], S[4 + (k & 1)], S[2 + k % 2])
        with torch.cuda.stream(si): dh[k].copy_(h[k*c:(k+1)*c], non_blocking=True)
        si.record_event(ev[k][0])
        if kind != "indep":
            sk.wait_event(ev[k][0])
            with torch.cuda.stream(sk): torch.cuda._sleep(200000)
            sk.record_event(ev[k][1]); so.wait_event(ev[k][1])
        with torch.cuda.stream(so): w[k*c:(k+1)*c].copy_(dw[k], non_blocking=True)
        so.record_event(ev[k][2])
        if kind == "indep": so.record_event(ev[k][1])
    torch.cuda.synchronize()
    print(kind)
    for k in range(N):
        print(f"chunk {k:2d}  h2d done {t0.elapsed_time(ev[k][0]):6.3f}  kernel done {t0.elapsed_time(ev[k][1]):6.3f}  d2h done {t0.elapsed_time(ev[k][2]):6.3f}")

def hostdriven(sleep):
    """D2H enqueued by the host once the chunk's kernel has finished, so no copy
    ever waits on an event inside a copy-engine queue."""
    evk = [torch.cuda.Event() for _ in range(N)]
    for k in range(N):
        with torch.cuda.stream(S[0]): dh[k].copy_(h[k*c:(k+1)*c], non_blocking=True)
        ev = torch.cuda.Event(); S[0].record_event(ev); S[4].wait_event(ev)
        with torch.cuda.stream(S[4]): torch.cuda._sleep(sleep)
        S[4].record_event(evk[k])
    for k in range(N):
        evk[k].synchronize()
        with torch.cuda.stream(S[2]): w[k*c:(k+1)*c].copy_(dw[k], non_blocking=True)

def aligned(sleep, lag=1):
    """D2H of chunk k also waits for the copy-in of chunk k + lag, so each D2H
    starts together with an H2D (in phase, as the independent copies run)."""
    eh = [torch.cuda.Event() for _ in range(N)]
    ek = [torch.cuda.Event() for _ in range(N)]
    for k in range(N + lag):
        if k < N:
            with torch.cuda.stream(S[0]): dh[k].copy_(h[k*c:(k+1)*c], non_blocking=True)
            S[0].record_event(eh[k]); S[4].wait_event(eh[k])
            with torch.cuda.stream(S[4]): torch.cuda._sleep(sleep)
            S[4].record_event(ek[k])
        j = k - lag
        if j >= 0:
            S[2].wait_event(ek[j])
            if k < N: S[2].wait_event(eh[k])
            with torch.cuda.stream(S[2]): w[j*c:(j+1)*c].copy_(dw[j], non_blocking=True)

for name, f in [("aligned lag1 sleep", lambda: aligned(200000)), ("aligned lag2 sleep", lambda: aligned(200000, 2)),
                ("aligned lag1 sleep=50k", lambda: aligned(50000))]:
    t = timeit(f)
    print(f"{name:24s} {t*1e3:6.2f} ms  {2*n/t/1e9:5.1f} GB/s", flush=True)
for name, f in [("host-driven sleep", lambda: hostdriven(200000)), ("host-driven sleep=50k", lambda: hostdriven(50000))]:
    t = timeit(f)
    print(f"{name:24s} {t*1e3:6.2f} ms  {2*n/t/1e9:5.1f} GB/s", flush=True)
