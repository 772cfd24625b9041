# NOTE: measured with an experimental patch that was not kept (see DESIGN.md 7d and
# profiles/short_r02.txt); the flags it uses no longer exist in the tree.
# A/B: weight boxes issued before griddepcontrol.wait (TIDAL_GEMM_PRE / _PREPF), warm rho = 1
mkdir -p gpurun_out/pre
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for rep in 1 2; do
for S in 256 867 2048; do
  for v in "0 0" "8 0" "8 16" "8 64"; do
    set -- $v
    TIDAL_GEMM_PRE=$1 TIDAL_GEMM_PREPF=$2 timeout 300 python tools/warm.py --seq $S --steps 10 --tag "S$S pre$1 pf$2" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], round(d['mean_ms'],3), round(d['median_ms'],3), d['token'])"
  done
done
done
