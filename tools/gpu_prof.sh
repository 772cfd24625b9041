#!/bin/bash
# ncu evidence: launch list (all kernels of one quick bench) + full captures of chosen kernels.
# KERNELS="<regex>@<skip>@<count> ..." (regex over demangled names)
mkdir -p gpurun_out
Q="--steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep"
if [ "${LAUNCH:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $Q > gpurun_out/ncu_launch.log 2>&1
fi
i=0
for spec in $KERNELS; do
  rx=${spec%%@*}; rest=${spec#*@}; skip=${rest%%@*}; cnt=${rest#*@}
  i=$((i+1))
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c $cnt -o gpurun_out/prof_$i -f python bench.py $Q > gpurun_out/ncu_$i.log 2>&1
done
ls -la gpurun_out
