mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu > gpurun_out/t5.log 2>&1; tail -12 gpurun_out/t5.log
TIDAL_FUSED_SHRINK=1 timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py tests/test_gpu_tp_local.py -q -m gpu -x > gpurun_out/t5f.log 2>&1; tail -3 gpurun_out/t5f.log
: > gpurun_out/ab5.jsonl
for rep in 1 2; do
for v in "TIDAL_FUSED_SHRINK=0" "TIDAL_FUSED_SHRINK=1"; do
  env TIDAL_GRAPH=0 $v timeout 300 python tools/warm.py --steps 10 --profile --tag "$v" 2>>gpurun_out/ab.err | tail -1 >> gpurun_out/ab5.jsonl
done
done
python - <<'P'
import json
for l in open("gpurun_out/ab5.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print(d["tag"], round(d["mean_ms"],2), round(d["min_ms"],2), d.get("gemm_us_per_launch"), d.get("kernels_ms_per_step", {}).get("lora_shrink"))
P
TIDAL_FUSED_SHRINK=1 TIDAL_GRAPH=0 TIDAL_GEMM_TRACE=20,0 TIDAL_GEMM_TRACE_FILE=gpurun_out/trace_qkv_p.bin timeout 300 python tools/warm.py --steps 2 --warmup 1 > /dev/null
python tools/gemm_trace.py gpurun_out/trace_qkv_p.bin 2>/dev/null | head -5
TIDAL_FUSED_SHRINK=1 TIDAL_GRAPH=0 TIDAL_GEMM_TRACE=20,3 TIDAL_GEMM_TRACE_FILE=gpurun_out/trace_down_p.bin timeout 300 python tools/warm.py --steps 2 --warmup 1 > /dev/null
python tools/gemm_trace.py gpurun_out/trace_down_p.bin 2>/dev/null | head -5
