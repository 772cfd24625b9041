# source-level ncu of the S = 256 QKV GEMM (who waits: producer on empty or MMA on full)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/q256
TIDAL_GRAPH=0 timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:gemm_tc_kernel<.int.1, .int.256, .int.2" -s 6 -c 1 -o gpurun_out/q256/qkv -f python tools/warm.py --seq 256 --steps 1 --warmup 1 > /dev/null 2>&1
ncu -i gpurun_out/q256/qkv.ncu-rep --page source --csv --print-source sass 2>/dev/null > gpurun_out/q256/src.csv
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/q256/src.csv')))
h=[r for r in rows if r and r[0]=='Address'][0]; si=h.index('Warp Stall Sampling (All Samples)')
ei=h.index('Instructions Executed') if 'Instructions Executed' in h else None
body=[r for r in rows if r and r[0].startswith('0x')]
tot=sum(float(r[si] or 0) for r in body)
for i,r in enumerate(sorted(body,key=lambda r:-float(r[si] or 0))[:14]):
    j=body.index(r)
    ctx=' | '.join(x[1][:40] for x in body[max(0,j-3):j])
    print(f"{float(r[si])/tot*100:5.1f}% exec {r[ei] if ei else ''}  {r[1][:60]}   <- {ctx}")
PY
