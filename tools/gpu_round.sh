#!/bin/bash
# One GPU session: tests, bench, ncu launch list and full captures.
set -x
mkdir -p gpurun_out
Q="--steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -q -m gpu > gpurun_out/gputests.log 2>&1
tail -4 gpurun_out/gputests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 600 gpurun_out/bench.json
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $Q > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 200 -c 4 -o gpurun_out/prof_gemm -f python bench.py $Q > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 45 -c 1 -o gpurun_out/prof_attn -f python bench.py $Q > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shrink_kernel -s 200 -c 2 -o gpurun_out/prof_shrink -f python bench.py $Q > gpurun_out/ncu_shrink.log 2>&1
fi
ls -la gpurun_out
