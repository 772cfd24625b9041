mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for d in 0 32 16; do
  TIDAL_TDIAG=$d TIDAL_FUSED_SHRINK=1 TIDAL_GRAPH=0 TIDAL_GEMM_TRACE=20,0 TIDAL_GEMM_TRACE_FILE=gpurun_out/trace_qkv_d$d.bin timeout 300 python tools/warm.py --steps 2 --warmup 1 | tail -1 | cut -c1-120
  echo "== QKV diag=$d"; python tools/gemm_trace.py gpurun_out/trace_qkv_d$d.bin | head -4 || true
done
