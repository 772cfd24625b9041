#!/bin/bash
# Round evidence under gpurun_out/prof/: the bench line, the ncu launch list of
# one quick bench (all kernels), ncu --set full captures of the prefill's top
# kernels and of the decode GEMVs, summaries and per-kernel DRAM traffic.
set -x
O=gpurun_out/prof
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
python tools/show_bench.py $O/bench.json
Q="--steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py $Q > $O/ncu_launch.log 2>&1
python tools/launches.py $O/launches.csv > $O/launches.txt
cat $O/launches.txt
i=0
for spec in "gemm_tc_kernel<.int.2,..int.128,..int.2@50@1" "gemm_tc_kernel<.int.1,..int.256@50@1" "gemm_tc_kernel<.int.3,..int.192@100@1" "gemm_tc_kernel<.int.3,..int.256@100@1" "attn_tc_kernel@100@1" "gemm_tc_kernel<.int.4@100@1" "shrink_reduce@100@1" "rmsnorm@100@1"; do
  rx=${spec%%@*}; rest=${spec#*@}; skip=${rest%%@*}; cnt=${rest#*@}
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c $cnt -o $O/prefill_$i -f python bench.py $Q > $O/ncu_$i.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:dec_|head_kernel" --csv --log-file $O/dec_launches.csv python tools/decode_prof.py --steps 4 > /dev/null 2>&1
python tools/launches.py $O/dec_launches.csv > $O/dec_launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:dec_gemv_kernel" -s 300 -c 4 -o $O/decode_gemv -f python tools/decode_prof.py --steps 4 > /dev/null 2>&1
for f in $O/*.ncu-rep; do python tools/ncu_summary.py $f; done > $O/ncu_full.txt 2>&1
ls -la $O
