# two-query-tile ping-pong attention: parity, per-op A/B, end-to-end A/B, ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k attention -x > gpurun_out/pp_tests.log 2>&1; tail -3 gpurun_out/pp_tests.log
grep -q "passed" gpurun_out/pp_tests.log && ! grep -q "failed" gpurun_out/pp_tests.log || { tail -40 gpurun_out/pp_tests.log; exit 1; }
for i in 1 2; do for a in 1 0; do echo "TIDAL_ATTN=$a"; TIDAL_ATTN=$a timeout 300 python tools/attn_bench.py --S 867 2048 8192; done; done
timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py tests/test_gpu_decode.py tests/test_gpu_tp_local.py -q -m gpu -x > gpurun_out/pp_e2e.log 2>&1; tail -3 gpurun_out/pp_e2e.log
for rep in 1 2; do for a in 1 0; do for S in 2048 8192; do
  TIDAL_ATTN=$a timeout 300 python tools/warm.py --seq $S --steps 10 --tag attn$a 2>/dev/null | tail -1
done; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_pp -c 1 -o gpurun_out/attn_pp python tools/attn_bench.py --S 2048 --reps 1 > gpurun_out/ncu_pp.log 2>&1
ncu -i gpurun_out/attn_pp.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[-1]
for k,x in zip(h,v):
  if k in ('gpu__time_duration.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','sm__issue_active.avg.pct_of_peak_sustained_elapsed'): print(k,x)"
