# half-width tail tiles (TIDAL_GEMM_HALF): parity + A/B (warm rho = 1, GEMM bench)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py tests/test_gpu_decode.py -q -x 2>&1 | tail -2
for r in 1 2; do for v in 1 0; do for S in 1154 2048; do
  TIDAL_GEMM_HALF=$v timeout 300 python tools/warm.py --seq $S --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('half', '$v', d['seq'], round(d['mean_ms'],3), round(d['median_ms'],3), d['token'])"
done; done; done
