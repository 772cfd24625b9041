# same-box A/B: ab/old (a previous commit, built) vs the working tree, warm rho=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for i in 1 2 3; do for side in old new; do
  d=$([ $side = old ] && echo ab/old || echo .)
  for S in ${AB_S:-2048 867 256}; do
    (cd $d && timeout 300 python tools/warm.py --seq $S --steps 10 --tag $side 2>/dev/null | tail -1) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], d['seq'], round(d['mean_ms'],2), round(d['min_ms'],2))"
  done
done; done
