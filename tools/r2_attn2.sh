mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k attention > gpurun_out/attn2_tests.log 2>&1; tail -5 gpurun_out/attn2_tests.log
for v in 1 0 1 0; do echo "v1=$v"; TIDAL_ATTN_V1=$v timeout 300 python tools/attn_bench.py --S 867 2048 8192; done
timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/attn2_e2e.log 2>&1; tail -3 gpurun_out/attn2_e2e.log
for v in 1 0; do TIDAL_ATTN_V1=$v timeout 300 python tools/warm.py --steps 10 --tag attnv1_$v | cut -c1-140; done
