#!/bin/bash
# One optimisation iteration on the GPU box: kernel/e2e parity, a bench line,
# then ncu --set full of the kernels named in KERNELS ("regex@skip@count ...").
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest ${TESTS:-tests/test_gpu_kernels.py tests/test_gpu_e2e.py} -q -m gpu -x > gpurun_out/gputests.log 2>&1
tail -3 gpurun_out/gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/show_bench.py gpurun_out/bench.json 2>/dev/null || tail -c 1500 gpurun_out/bench.json
Q="--steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep"
i=0
for spec in $KERNELS; do
  rx=${spec%%@*}; rest=${spec#*@}; skip=${rest%%@*}; cnt=${rest#*@}
  i=$((i+1))
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c $cnt -o gpurun_out/prof_$i -f python bench.py $Q > gpurun_out/ncu_$i.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_$i.ncu-rep
done
