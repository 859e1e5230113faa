"""Probe the GPU box: host cores/RAM, pinned H2D/D2H bandwidth, pinned-alloc speed."""
import os, time, json, subprocess
import torch
out = {}
out["cpu_count"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().split("\n")[:3]
out["gpu"] = torch.cuda.get_device_name(0)
p = torch.cuda.get_device_properties(0)
out["sms"] = p.multi_processor_count
out["total_mem"] = p.total_memory
for mb in (17, 64, 256, 1024):
    n = mb * 2**20
    t0 = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    out[f"pin_alloc_{mb}MB_s"] = time.time() - t0
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    out[f"h2d_{mb}MB_GBs"] = n * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            h.copy_(d, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    out[f"d2h_{mb}MB_GBs"] = n * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    del h, d
# big pinned alloc time
t0 = time.time()
h = torch.empty(8 * 2**30, dtype=torch.uint8, pin_memory=True)
out["pin_alloc_8GB_s"] = time.time() - t0
del h
out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,pcie.link.gen.current,pcie.link.width.current,clocks.sm,clocks.max.sm", "--format=csv"], capture_output=True, text=True).stdout
out["lscpu"] = subprocess.run(["bash", "-c", "lscpu | head -20"], capture_output=True, text=True).stdout
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
