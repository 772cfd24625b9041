# ncu launch list of one quick bench with the final round-2 kernels
O=gpurun_out/prof3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
Q="--steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep --decode-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py $Q > $O/ncu_launch.log 2>&1
python tools/launches.py $O/launches.csv > $O/launches.txt; cat $O/launches.txt
