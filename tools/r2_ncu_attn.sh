O=gpurun_out/prof2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
Q="--steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep --decode-steps 0"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:attn_pp_kernel" -s 100 -c 1 -o $O/prefill_4 -f python bench.py $Q > $O/ncu_4.log 2>&1
python tools/ncu_summary.py $O/prefill_4.ncu-rep
