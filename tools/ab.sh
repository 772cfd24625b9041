#!/bin/bash
# Same-box A/B of two library builds: ab/old (a previous commit, built in
# place) vs the working tree; alternating bench runs, warm (rho = 1) and
# Eq. 1 TTFT.  Usage: bash tools/ab.sh [rounds]
R=${1:-2}
mkdir -p gpurun_out
for i in $(seq $R); do
  for side in old new; do
    d=$([ $side = old ] && echo ab/old || echo .)
    (cd $d && timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep 2>/dev/null | tail -1) > gpurun_out/ab_${side}_$i.json
    python - "$side" gpurun_out/ab_${side}_$i.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read())
k = d["kernels"]
print(sys.argv[1], "ttft", round(d["value"], 2), "warm", round(d["sweep_ms"]["warm_rho1"], 2),
      "shrink", round(k["lora_shrink"]["ms_per_step"], 2), "attn", round(k["attention"]["ms_per_step"], 2),
      "clk", d["clocks"]["sm_mhz"])
PY
  done
done
