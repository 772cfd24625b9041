# refresh the shape sweep with the final round-2 kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
rm -f gpurun_out/sweep_r02.jsonl
timeout 1800 python tools/sweep.py --out gpurun_out/sweep_r02.jsonl > gpurun_out/sweep_r02.log 2>&1; tail -2 gpurun_out/sweep_r02.log
timeout 900 python tools/sweep.py --config 7b --out gpurun_out/sweep_r02.jsonl >> gpurun_out/sweep_r02.log 2>&1
timeout 900 python tools/sweep.py --S 512 1154 4096 --rho 1.0 --out gpurun_out/sweep_r02.jsonl >> gpurun_out/sweep_r02.log 2>&1
python - <<'P'
import json
for l in open("gpurun_out/sweep_r02.jsonl"):
    d=json.loads(l); print(d["config"], d["S"], d["lora_rank"], d["rho_requested"], round(d["ttft_ms"],2), "roof", round(d["roof_ms"],2), d["bound"], "frac", round(d["frac"],3))
P
