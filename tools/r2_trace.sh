mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for v in 0 1; do
  TIDAL_FUSED_SHRINK=$v TIDAL_GRAPH=0 TIDAL_GEMM_TRACE=20,0 TIDAL_GEMM_TRACE_FILE=gpurun_out/trace_qkv_f$v.bin timeout 300 python tools/warm.py --steps 2 --warmup 1 | tail -1
  echo "== QKV fused=$v"; python tools/gemm_trace.py gpurun_out/trace_qkv_f$v.bin
  TIDAL_FUSED_SHRINK=$v TIDAL_GRAPH=0 TIDAL_GEMM_TRACE=20,3 TIDAL_GEMM_TRACE_FILE=gpurun_out/trace_down_f$v.bin timeout 300 python tools/warm.py --steps 2 --warmup 1 | tail -1
  echo "== down fused=$v"; python tools/gemm_trace.py gpurun_out/trace_down_f$v.bin
done
