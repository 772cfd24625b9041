mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k attention > gpurun_out/attn3_tests.log 2>&1; tail -3 gpurun_out/attn3_tests.log
for i in 1 2; do for side in old new; do d=$([ $side = old ] && echo ab/old || echo .); echo $side; (cd $d && timeout 300 python tools/attn_bench.py --S 867 2048 8192); done; done
TIDAL_ATTN_TRACE=gpurun_out/attn_trace3.bin timeout 300 python tools/attn_bench.py --S 8192 --reps 1 > /dev/null; python tools/attn_trace.py gpurun_out/attn_trace3.bin
timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py tests/test_gpu_decode.py -q -m gpu -x > gpurun_out/attn3_e2e.log 2>&1; tail -3 gpurun_out/attn3_e2e.log
AB_S="2048 8192" bash tools/r2_ab_warm.sh 2>&1 | head -8
