# A/B of kernel variants at warm rho=1 (13B, S=2048, r16): one process each, interleaved
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
: > gpurun_out/ab.jsonl
for rep in 1 2; do
for v in "TIDAL_FUSED_SHRINK=0" "TIDAL_FUSED_SHRINK=1" "TIDAL_TDIAG=1" "TIDAL_RESID_SPLIT=1" ; do
  env $v timeout 300 python tools/warm.py --steps 10 --tag "$v" ${WARM_ARGS} 2>>gpurun_out/ab.err | tail -1 >> gpurun_out/ab.jsonl
done
done
python - <<'P'
import json
for l in open("gpurun_out/ab.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print(d["tag"], round(d["mean_ms"],2), round(d["min_ms"],2), d.get("gemm_us_per_launch"))
P
timeout 600 python tools/gemm_bench.py --resid-sweep --reps 20 > gpurun_out/resid_sweep.txt 2>&1; tail -40 gpurun_out/resid_sweep.txt
