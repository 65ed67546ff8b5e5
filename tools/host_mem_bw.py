"""Host DRAM bandwidth of the box (development aid, quoted in DESIGN.md §6):
numpy copies of 1 GiB pinned-size buffers on T threads (numpy releases the GIL),
read + write bytes / time; and the sum of N concurrent pinned H2D+D2H streams
is bounded by it."""
import os, sys, threading, time
import numpy as np

def run(T, nbytes=1 << 30, reps=3):
    srcs = [np.ones(nbytes // 8 // T) for _ in range(T)]
    dsts = [np.empty_like(s) for s in srcs]
    def work(i):
        for _ in range(reps):
            np.copyto(dsts[i], srcs[i])
    for i in range(T):
        work(i)  # warm
    ts = [threading.Thread(target=work, args=(i,)) for i in range(T)]
    t0 = time.perf_counter()
    for t in ts: t.start()
    for t in ts: t.join()
    dt = time.perf_counter() - t0
    return 2 * nbytes * reps / dt / 1e9

cores = os.cpu_count()
for T in (1, 4, 8, cores):
    print(f"host DRAM copy, {T:2d} threads: {run(T):6.1f} GB/s (read + write)", flush=True)
