mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
: > gpurun_out/ab2.jsonl
for v in "TIDAL_FUSED_SHRINK=0" "TIDAL_FUSED_SHRINK=1" "TIDAL_TDIAG=2" "TIDAL_FUSED_SHRINK=0" "TIDAL_FUSED_SHRINK=1" "TIDAL_TDIAG=2"; do
  env $v timeout 300 python tools/warm.py --steps 10 --profile --tag "$v" 2>>gpurun_out/ab.err | tail -1 >> gpurun_out/ab2.jsonl
done
python - <<'P'
import json
for l in open("gpurun_out/ab2.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print(d["tag"], round(d["mean_ms"],2), round(d["min_ms"],2), d.get("gemm_us_per_launch"))
P
for v in 0 1; do
TIDAL_FUSED_SHRINK=$v timeout 600 ncu --set full --clock-control none --import-source on -k "regex:gemm_tc_kernel<1" -s 45 -c 1 -o gpurun_out/qkv_fused$v -f python tools/warm.py --steps 1 --warmup 1 > gpurun_out/ncu_q$v.log 2>&1
python tools/ncu_summary.py gpurun_out/qkv_fused$v.ncu-rep 2>&1 | head -20
done
