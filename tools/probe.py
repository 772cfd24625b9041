"""Hardware probe on the GPU box: PCIe H2D bandwidth from pinned host memory
(the roofline denominator B_h2d), topology, host cores."""
import json
import os
import subprocess
import time

import torch


def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)


def h2d(nbytes, reps=10, chunk=None):
    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    src.fill_(1)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = 0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            if chunk:
                for o in range(0, nbytes, chunk):
                    dst[o:o + chunk].copy_(src[o:o + chunk], non_blocking=True)
            else:
                dst.copy_(src, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


out = {"cpu": sh("lscpu | head -20"), "nproc": os.cpu_count(),
       "affinity": len(os.sched_getaffinity(0)),
       "numa": sh("ls /sys/devices/system/node | grep node"),
       "smi": sh("nvidia-smi --query-gpu=name,pci.bus_id,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,clocks.sm,clocks.max.sm --format=csv"),
       "topo": sh("nvidia-smi topo -m"), "mem": sh("free -g")}
bus = torch.cuda.get_device_properties(0)
out["h2d_GBps"] = {str(n): h2d(n) for n in (64 << 20, 256 << 20, 1 << 30)}
out["h2d_1GiB_chunk64MB"] = h2d(1 << 30, chunk=64 << 20)
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    a @ a
torch.cuda.synchronize()
t = time.time()
for _ in range(10):
    a @ a
torch.cuda.synchronize()
out["bf16_tflops"] = 10 * 2 * 8192 ** 3 / (time.time() - t) / 1e12
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
print(json.dumps({k: out[k] for k in ("h2d_GBps", "h2d_1GiB_chunk64MB", "bf16_tflops", "nproc", "affinity")}))
print(out["smi"]); print(out["topo"][:2000]); print(out["cpu"][:600]); print(out["numa"], out["mem"])
