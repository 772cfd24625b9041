# GEMM tail prefetch of the next GEMM's weights (TIDAL_GEMM_PF): parity + same-box A/B, warm rho = 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py tests/test_gpu_tp_local.py -q -x 2>&1 | tail -1
for r in 1 2; do for S in 256 867 2048; do for v in 1 0; do
  TIDAL_GEMM_PF=$v timeout 300 python tools/warm.py --seq $S --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf', '$v', d['seq'], round(d['mean_ms'],3), round(d['median_ms'],3), d['token'])"
done; done; done
