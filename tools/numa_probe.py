"""Host NUMA placement vs PCIe copy bandwidth (development aid): for every NUMA
node whose CPUs this process may run on, bind to it, allocate pinned buffers
(first touch) and time H2D, D2H and both at once."""
import os, glob, torch

def cpus_of(node):
    s = open(f"/sys/devices/system/node/node{node}/cpulist").read().strip()
    out = set()
    for part in s.split(","):
        if not part: continue
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out

allowed = os.sched_getaffinity(0)
nodes = sorted(int(p.rsplit("node", 1)[1]) for p in glob.glob("/sys/devices/system/node/node[0-9]*"))
print("allowed cpus", sorted(allowed), "nodes", nodes, flush=True)
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    bus = pynvml.nvmlDeviceGetPciInfo(h).busId
    bus = bus.decode() if isinstance(bus, bytes) else bus
    short = bus[-12:].lower()
    print("gpu0 pci", bus, "numa_node", open(f"/sys/bus/pci/devices/{short}/numa_node").read().strip(), flush=True)
    try:
        n = (os.cpu_count() + 63) // 64
        print("nvml ideal cpu mask", [hex(x) for x in pynvml.nvmlDeviceGetCpuAffinity(h, n)], flush=True)
    except Exception as e:
        print("nvml affinity:", e)
except Exception as e:
    print("nvml:", e)
N = 256 << 20
d_in = torch.empty(N, dtype=torch.uint8, device="cuda"); d_out = torch.empty_like(d_in)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bw(fn, reps=8):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); b.record(); torch.cuda.synchronize()
    return N * reps / a.elapsed_time(b) / 1e6
for node in nodes:
    c = cpus_of(node) & allowed
    if not c:
        print(f"node {node}: no allowed cpus"); continue
    os.sched_setaffinity(0, c)
    hi = torch.empty(N, dtype=torch.uint8).pin_memory(); ho = torch.empty(N, dtype=torch.uint8).pin_memory()
    hi.fill_(1); ho.fill_(2)
    def both():
        with torch.cuda.stream(s1): d_in.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2): ho.copy_(d_out, non_blocking=True)
    print(f"node {node} ({len(c)} cpus): h2d {bw(lambda: d_in.copy_(hi, non_blocking=True)):.1f}  d2h {bw(lambda: ho.copy_(d_out, non_blocking=True)):.1f}  "
          f"both {2 * bw(both):.1f} GB/s", flush=True)
    del hi, ho
os.sched_setaffinity(0, allowed)
