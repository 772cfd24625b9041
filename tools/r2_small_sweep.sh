# every (bn, cg, split-K) GEMM variant at the short-prompt shapes (planner check)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/small
for S in 256 512 867 1154; do
  timeout 600 python tools/gemm_bench.py --S $S --small-sweep --reps 10 > gpurun_out/small/S$S.txt 2>&1
  echo "== S=$S"; cat gpurun_out/small/S$S.txt
  timeout 300 python tools/warm.py --seq $S --steps 5 --profile --tag S$S | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warm', d['seq'], round(d['mean_ms'],2), d['gemm_us_per_launch'])"
done
