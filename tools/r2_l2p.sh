# residual stream X as persisting L2 lines (TIDAL_L2_PERSIST): warm rho = 1, same box, interleaved
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for r in 1 2 3 4; do for S in 2048 867; do for v in 1 0; do
  TIDAL_L2_PERSIST=$v timeout 300 python tools/warm.py --seq $S --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S', d['seq'], 'persist', '$v', round(d['mean_ms'],3), round(d['median_ms'],3), d['token'])"
done; done; done
