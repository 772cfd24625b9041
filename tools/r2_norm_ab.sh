# persistent RMSNorm: same-box A/B against HEAD (ab/old), warm rho = 1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "rmsnorm" 2>&1 | tail -1
for r in 1 2 3; do for S in 256 2048; do
  timeout 300 python tools/warm.py --seq $S --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', d['seq'], round(d['mean_ms'],3), d['token'])"
  (cd ab/old && timeout 300 python tools/warm.py --seq $S --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['seq'], round(d['mean_ms'],3), d['token'])")
done; done
