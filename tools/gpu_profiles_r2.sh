#!/bin/bash
# Round-2 evidence under gpurun_out/prof2/: ncu launch list of one quick bench,
# ncu --set full captures of the prefill's top kernels, per-kernel summaries,
# then compute-sanitizer over the tiny / hd-128 workload.
O=gpurun_out/prof2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { cat $O/build.log; exit 1; }
Q="--steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep --decode-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py $Q > $O/ncu_launch.log 2>&1
python tools/launches.py $O/launches.csv > $O/launches.txt
cat $O/launches.txt
i=0
for spec in "gemm_tc_kernel<.int.2, .int.128, .int.2@50@1" "gemm_tc_kernel<.int.1, .int.256, .int.2@50@1" "gemm_tc_kernel<.int.3, .int.256, .int.2@100@2" "attn_pp_kernel@100@1" "rmsnorm@100@1" "lora_pack@40@1" "head_kernel@2@1"; do
  rx=${spec%%@*}; rest=${spec#*@}; skip=${rest%%@*}; cnt=${rest#*@}
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c $cnt -o $O/prefill_$i -f python bench.py $Q > $O/ncu_$i.log 2>&1
done
for f in $O/*.ncu-rep; do python tools/ncu_summary.py $f; done > $O/ncu_full.txt 2>&1
grep -E "ncu-rep|time_duration|dram__bytes_read|dram__bytes_write|tensor_cycles" $O/ncu_full.txt
# compute-sanitizer runs (tools/sanitize.sh) are no longer allowed on the pool; the
# round-2 logs under profiles/sanitizer_r02/ come from before that
ls -la $O
