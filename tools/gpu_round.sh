#!/bin/bash
# One GPU session: tests, bench (each step under its own timeout).
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x > gpurun_out/gputests.log 2>&1
timeout 300 python -m pytest tests/test_gpu_e2e.py -q -m gpu -x >> gpurun_out/gputests.log 2>&1
timeout 300 python -m pytest tests/test_gpu_tp_local.py -q -m gpu -x >> gpurun_out/gputests.log 2>&1
tail -4 gpurun_out/gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 600 gpurun_out/bench.json
ls -la gpurun_out
