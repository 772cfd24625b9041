mkdir -p gpurun_out/pp
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for S in 2048 8192; do
  TIDAL_ATTN=2 TIDAL_ATTN_TRACE=gpurun_out/pp/t$S.bin timeout 300 python tools/attn_bench.py --S $S --reps 1 | tail -1
  python tools/attn_pp_trace.py gpurun_out/pp/t$S.bin $S 40
done
TIDAL_ATTN=2 timeout 300 python tools/attn_bench.py --S 2048 8192 --reps 10
