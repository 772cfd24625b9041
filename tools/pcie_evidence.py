"""PCIe evidence for the streaming path: while a 13B template at rho = 0
streams 26 GB per invocation (10 invocations back to back), sample the
device's PCIe counters with `nvidia-smi dmon -s t` (rxpci = host->device
MB/s, once per second) and report them beside the event-timed H2D rate.

    python tools/pcie_evidence.py > gpurun_out/pcie.txt
"""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2503_06421_b200 import build  # noqa: E402

build.build()
from paper_2503_06421_b200 import tidal as T  # noqa: E402

cfg = synth.config("13b")
tensors, fill = synth.model_inputs(cfg, 0)
model = T.Model(bench.cfg_dict(cfg), tensors, "base:0", fill=fill)
tpl = T.Template(model, T.Trace(model), T.template_opts(resident_bytes=0, max_tokens=2048, device=0))
tok = synth.prompt_fast(cfg, 2048, 0)
tpl.invoke(tok, want_logits=False)  # warm
dmon = subprocess.Popen(["nvidia-smi", "dmon", "-s", "t", "-d", "1", "-i", "0"],
                        stdout=subprocess.PIPE, text=True)
time.sleep(1.5)
rates = []
t0 = time.time()
for _ in range(10):
    _, _, st = tpl.invoke(tok, want_logits=False)
    rates.append((st["bytes_streamed"] + st["bytes_adapter"]) / ((st["h2d_last_ms"] - st["h2d_first_ms"]) / 1e3) / 1e9)
elapsed = time.time() - t0
time.sleep(1.5)
dmon.terminate()
out = dmon.communicate()[0]
print("# event-timed H2D per invocation (GB/s):", " ".join(f"{r:.1f}" for r in rates))
print(f"# 10 invocations x {st['bytes_streamed'] / 1e9:.2f} GB in {elapsed:.2f} s wall")
print("# nvidia-smi dmon -s t (rxpci/txpci in MB/s, 1 s samples):")
print(out)
