mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
: > gpurun_out/ab4.jsonl
for rep in 1 2; do
for v in "TIDAL_FUSED_SHRINK=0" "TIDAL_FUSED_SHRINK=1 TIDAL_FUSE_MASK=5" "TIDAL_FUSED_SHRINK=1 TIDAL_FUSE_MASK=5 TIDAL_TPAD=256" "TIDAL_FUSED_SHRINK=1 TIDAL_FUSE_MASK=5 TIDAL_TPAD=128" "TIDAL_FUSED_SHRINK=1 TIDAL_TPAD=256"; do
  env TIDAL_GRAPH=0 $v timeout 300 python tools/warm.py --steps 10 --profile --tag "$v" 2>>gpurun_out/ab.err | tail -1 >> gpurun_out/ab4.jsonl
done
done
python - <<'P'
import json
for l in open("gpurun_out/ab4.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print(d["tag"], round(d["mean_ms"],2), round(d["min_ms"],2), d.get("gemm_us_per_launch"), d.get("kernels_ms_per_step", {}).get("lora_shrink"))
P
