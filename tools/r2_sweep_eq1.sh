# TTFT at Eq. 1 (adapter counted) across prompt lengths, 13B r16 and 7B (paper fig:ttft-len analog)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
rm -f gpurun_out/sweep_eq1.jsonl
timeout 1800 python tools/sweep.py --eq1 --out gpurun_out/sweep_eq1.jsonl > gpurun_out/sweep_eq1.log 2>&1
timeout 900 python tools/sweep.py --eq1 --config 7b --S 256 2048 8192 --out gpurun_out/sweep_eq1.jsonl >> gpurun_out/sweep_eq1.log 2>&1
python - <<'P'
import json
for l in open("gpurun_out/sweep_eq1.jsonl"):
    d=json.loads(l); print(d["config"], d["S"], "rho", round(d["rho_realized"],3), "ttft", round(d["ttft_ms"],2), "warm", round(d["t_warm_ms"],2), "roof", round(d["roof_ms"],2), d["bound"], "f", round(d["frac"],3), "ttft/warm", round(d["ttft_ms"]/d["t_warm_ms"],3))
P
