#!/bin/bash
# ncu evidence: launch list (all kernels of one quick bench) + full captures of chosen kernels.
mkdir -p gpurun_out
Q="--steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $Q > gpurun_out/ncu_launch.log 2>&1
for spec in $KERNELS; do
  name=${spec%%:*}; rest=${spec#*:}; skip=${rest%%:*}; cnt=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c $cnt -o gpurun_out/prof_$name -f python bench.py $Q > gpurun_out/ncu_$name.log 2>&1
done
ls -la gpurun_out
