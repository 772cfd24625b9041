# paired-tile attention, single-pass softmax: parity, A/B vs single tiles, ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "attention or head" -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_e2e.py -q -m gpu -x -k "batch" 2>&1 | tail -2
for i in 1 2; do for a in 1 2; do echo "TIDAL_ATTN=$a"; TIDAL_ATTN=$a timeout 300 python tools/attn_bench.py --S 867 1154 2048 4096 8192; done; done
TIDAL_ATTN=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_pp -c 1 -o gpurun_out/attn_pp3 python tools/attn_bench.py --S 2048 --reps 1 > gpurun_out/ncu_pp3.log 2>&1
ncu -i gpurun_out/attn_pp3.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[-1]
for k,x in zip(h,v):
  if k in ('gpu__time_duration.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','sm__issue_active.avg.pct_of_peak_sustained_elapsed'): print(k,x)"
