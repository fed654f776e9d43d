"""One-off probe of the GPU box: host cores/RAM, pinned host<->device link GB/s."""
import os, subprocess, json, time
import torch

out = {}
out["cpu_count"] = os.cpu_count()
try:
    out["lscpu_model"] = [l for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines() if "Model name" in l]
except Exception as e:
    out["lscpu_model"] = str(e)
with open("/proc/meminfo") as f:
    out["meminfo"] = [l.strip() for l in f.readlines()[:3]]
out["gpu"] = torch.cuda.get_device_name(0)
p = torch.cuda.get_device_properties(0)
out["sms"] = p.multi_processor_count
out["hbm_gib"] = p.total_memory / 2**30
for mib in (16, 64, 256):
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                fn()
            e1.record(s)
        e1.synchronize()
        out[f"{name}_{mib}MiB_GBs"] = n * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    # bidirectional concurrently
    s2 = torch.cuda.Stream()
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    out[f"bidir_{mib}MiB_GBs_each"] = n * 10 / (time.perf_counter() - t0) / 1e9
# pinned alloc time for 4 GiB
t0 = time.perf_counter()
big = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
out["pin_alloc_4GiB_s"] = time.perf_counter() - t0
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
