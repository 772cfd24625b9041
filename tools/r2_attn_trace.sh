mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for S in 2048 8192; do
  TIDAL_ATTN_TRACE=gpurun_out/attn_trace_$S.bin timeout 300 python tools/attn_bench.py --S $S --reps 1
  python tools/attn_trace.py gpurun_out/attn_trace_$S.bin
done
