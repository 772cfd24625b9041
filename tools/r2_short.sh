mkdir -p gpurun_out/short
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for S in 256 867 1154 2048; do timeout 300 python tools/warm.py --seq $S --steps 10 --profile --tag S$S | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['seq'], round(d['mean_ms'],2), d['gemm_us_per_launch'])"; done
timeout 600 python tools/gemm_bench.py --S 256 --small-sweep --reps 10 > gpurun_out/short/small256.txt 2>&1; cat gpurun_out/short/small256.txt
TIDAL_GRAPH=0 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemm_tc_kernel<.int.(1|2)" -s 20 -c 2 -o gpurun_out/short/qkv_gu_256 -f python tools/warm.py --seq 256 --steps 1 --warmup 1 > gpurun_out/short/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/short/qkv_gu_256.ncu-rep
