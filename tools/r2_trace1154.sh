# QKV / gate-up GEMM timelines at S = 1154 (runtime) vs the standalone rate
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/tr
for gm in 0 2; do
  TIDAL_GRAPH=0 TIDAL_GEMM_TRACE=20,$gm TIDAL_GEMM_TRACE_FILE=gpurun_out/tr/t$gm.bin timeout 300 python tools/warm.py --seq 1154 --steps 2 --warmup 1 > /dev/null 2>&1
  echo "== gemm $gm"; python tools/gemm_trace.py gpurun_out/tr/t$gm.bin
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tr/l.csv python tools/warm.py --seq 1154 --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/tr/l.csv | head -12
