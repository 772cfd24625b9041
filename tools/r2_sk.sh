mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tools/sk_repro.py > gpurun_out/sk_memcheck.txt 2>&1; tail -15 gpurun_out/sk_memcheck.txt
timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py tests/test_gpu_kernels.py tests/test_gpu_tp_local.py -q -m gpu -x > gpurun_out/sk_tests.log 2>&1; tail -4 gpurun_out/sk_tests.log
: > gpurun_out/sk_ab.txt
for rep in 1 2; do for v in 0 1; do for S in 2048 867 256; do
  TIDAL_STREAMK=$v timeout 300 python tools/warm.py --seq $S --steps 10 --tag sk$v 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], d['seq'], round(d['mean_ms'],2), round(d['min_ms'],2))" | tee -a gpurun_out/sk_ab.txt
done; done; done
TIDAL_GRAPH=0 TIDAL_GEMM_TRACE=20,0 TIDAL_GEMM_TRACE_FILE=gpurun_out/trace_qkv_sk.bin timeout 300 python tools/warm.py --steps 2 --warmup 1 > /dev/null
python tools/gemm_trace.py gpurun_out/trace_qkv_sk.bin 2>/dev/null | head -6
