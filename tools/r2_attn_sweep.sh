mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
TIDAL_ATTN_SPLIT=4 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k attention > gpurun_out/attn4_tests.log 2>&1; tail -3 gpurun_out/attn4_tests.log
for sp in 2 4 2 4; do echo "split $sp"; TIDAL_ATTN_SPLIT=$sp timeout 300 python tools/attn_bench.py --S 867 2048 8192; done
for sp in 2 4; do TIDAL_ATTN_SPLIT=$sp timeout 300 python tools/warm.py --steps 10 --tag split$sp | cut -c1-160; done
timeout 1500 python tools/sweep.py --S 256 867 1154 2048 4096 8192 --rho 1.0 --out gpurun_out/sweep_short.jsonl > gpurun_out/sweep_short.log 2>&1
python - <<'P'
import json
for l in open("gpurun_out/sweep_short.jsonl"):
    d=json.loads(l); print(d["S"], d["rho_requested"], round(d["ttft_ms"],2), "roof", round(d["roof_ms"],2), d["bound"], "frac", round(d["frac"],3))
P
for S in 256 867; do timeout 300 python tools/warm.py --seq $S --steps 10 --profile --tag S$S; done
