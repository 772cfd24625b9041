# two TMA producer threads per GEMM CTA (A side / B side) vs one (TIDAL_GEMM_P1=1): parity + same-box A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
for r in 1 2; do for S in 256 867 2048; do for v in 0 1; do
  TIDAL_GEMM_P1=$v timeout 300 python tools/warm.py --seq $S --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('p1', '$v', d['seq'], round(d['mean_ms'],3), round(d['median_ms'],3), d['token'])"
done; done; done
