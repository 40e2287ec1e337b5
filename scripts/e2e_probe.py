"""Where the e2e step goes (development tool): host enqueue time per
HostPipeline.submit, the pipelined step time, and the PCIe copy rates alone
(pinned 7.08 MB D2H, 2.6 MB H2D) on configs[1]."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
from paper_2512_06443_b200.pipeline import HostPipeline  # noqa: E402

dev = torch.device("cuda")
M, K, N, g = 6912, 2560, 256, 4
W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
pw = v.pack_weights_device(W, g)
x = np.random.default_rng(0).standard_normal((K, N)).astype(np.float32)
for depth in (2, 3, 4):
    pipe = HostPipeline(pw, synth.W_SCALE, K, N, dev, depth=depth)
    xp = [torch.from_numpy(x).pin_memory() for _ in range(depth)]
    op = [torch.empty((M, N), dtype=torch.float32).pin_memory() for _ in range(depth)]
    for i in range(8):
        pipe.submit(xp[i % depth], op[i % depth])
    pipe.synchronize()
    for steps in (20, 200):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(pipe.s_in)
        for i in range(steps):
            pipe.submit(xp[i % depth], op[i % depth])
        t1 = time.perf_counter()
        pipe.s_out.wait_stream(pipe.s_in)
        pipe.s_out.wait_stream(pipe.s_cmp)
        b.record(pipe.s_out)
        torch.cuda.synchronize()
        print(f"depth {depth} steps {steps}: host enqueue {(t1 - t0) / steps * 1e6:7.1f} us/step, "
              f"device {a.elapsed_time(b) / steps * 1e3:7.1f} us/step", flush=True)
d_out = torch.empty((M, N), device=dev)
h_out = torch.empty((M, N)).pin_memory()
d_in = torch.empty((K, N), device=dev)
h_in = torch.from_numpy(x).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("D2H 7.08 MB", lambda: h_out.copy_(d_out, non_blocking=True)),
                 ("H2D 2.62 MB", lambda: d_in.copy_(h_in, non_blocking=True))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 50
    nb = (M * N * 4) if name.startswith("D2H") else (K * N * 4)
    print(f"{name}: {ms * 1e3:7.1f} us ({nb / ms / 1e6:6.1f} GB/s)")
# both directions at once (full duplex?)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record()
with torch.cuda.stream(s1):
    for _ in range(50):
        h_out.copy_(d_out, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(50):
        d_in.copy_(h_in, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
b.record()
torch.cuda.synchronize()
print(f"D2H + H2D concurrently: {a.elapsed_time(b) / 50 * 1e3:7.1f} us per pair")

# ---- NUMA placement of the pinned buffers: the GPU's own node vs elsewhere
props = torch.cuda.get_device_properties(dev)
bdf = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
base = f"/sys/bus/pci/devices/{bdf}"
node = open(f"{base}/numa_node").read().strip() if os.path.exists(f"{base}/numa_node") else "?"
cpus = open(f"{base}/local_cpulist").read().strip() if os.path.exists(f"{base}/local_cpulist") else "?"
print(f"GPU {bdf}: numa_node {node}, local_cpulist {cpus}; nodes online "
      f"{open('/sys/devices/system/node/online').read().strip()}; process affinity {len(os.sched_getaffinity(0))} cpus")


def parse(lst):
    out = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def copy_rates(tag):
    h_in2 = torch.from_numpy(x).pin_memory()
    h_out2 = torch.empty((M, N)).pin_memory()
    for name, fn, nb in (("D2H", lambda: h_out2.copy_(d_out, non_blocking=True), M * N * 4),
                         ("H2D", lambda: d_in.copy_(h_in2, non_blocking=True), K * N * 4)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 50
        print(f"  {tag} {name}: {ms * 1e3:7.1f} us ({nb / ms / 1e6:6.1f} GB/s)", flush=True)


if cpus != "?":
    local = parse(cpus)
    allc = os.sched_getaffinity(0)
    copy_rates("default affinity")
    os.sched_setaffinity(0, local & allc or allc)
    copy_rates("GPU-local cpus")
    other = allc - local
    if other:
        os.sched_setaffinity(0, other)
        copy_rates("remote cpus")
    os.sched_setaffinity(0, allc)
