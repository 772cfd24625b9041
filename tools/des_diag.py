import json, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import synth
from paper_2503_06421_b200 import build
build.build()
from paper_2503_06421_b200 import tidal as T
cfg = synth.config("13b"); S, r = 2048, 16
cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab, rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
tensors, fill = synth.model_inputs(cfg, 0)
model = T.Model(cd, tensors, "base:0", fill=fill)
tpl = T.Template(model, T.Trace(model), T.template_opts(resident_bytes=0, max_tokens=S, device=0))
slots, nb = tpl.adapter_layout(r, 0x7F); buf = T.PinnedBuffer(nb); synth.adapter_fill(cfg, r, 1, slots, buf.view(), 0x7F)
tok = synth.prompt_fast(cfg, S, 0)
def run(dbg):
    tpl.set_debug(dbg | T.DEBUG_SCRUB_L2)
    ad = T.Adapter(tpl, r, 1.0, 0x7F, buf, nb, "adapter:1")
    _, _, st = tpl.invoke(tok, ad, want_logits=False)
    return st
st0 = run(T.DEBUG_SERIAL)
b = (st0["bytes_streamed"] + st0["bytes_adapter"]) / ((st0["h2d_last_ms"] - st0["h2d_first_ms"]) / 1e3)
tpl.resize(T.template_opts(resident_bytes=T.U64_MAX))
for _ in range(3): stw = run(T.DEBUG_TIMELINE)
tlw = tpl.timeline()
dw = np.diff(np.append(tlw["op_start_ms"], tlw["end_ms"]))
tpl.resize(T.template_opts(eq1=True, t_ttft_s=stw["device_ms"] / 1e3, b_pcie_Bps=b))
for _ in range(2): sts = run(T.DEBUG_TIMELINE)
tls = tpl.timeline()
ds = np.diff(np.append(tls["op_start_ms"], tls["end_ms"]))
n = len(dw)
print("warm", stw["device_ms"], "stream", sts["device_ms"], "ops", n)
diff = ds - dw
idx = np.argsort(-diff)[:15]
for i in sorted(idx):
    print(f"op {i:4d} warm {dw[i]*1e3:8.1f} us  stream {ds[i]*1e3:8.1f} us  start {tls['op_start_ms'][i]:7.2f}")
# cumulative by decile
for q in range(10):
    a, bq = q * n // 10, (q + 1) * n // 10
    print(f"ops {a}-{bq}: warm {dw[a:bq].sum():6.2f} ms stream {ds[a:bq].sum():6.2f} ms")
print("group ends", np.round(np.sort(tls["group_end_ms"])[-6:], 2))
