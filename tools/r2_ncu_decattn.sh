python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/dec
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dec_attn -s 40 -c 1 -o gpurun_out/dec/attn -f python tools/decode_prof.py --steps 2 > /dev/null 2>&1
ncu -i gpurun_out/dec/attn.ncu-rep --page details --csv 2>/dev/null | grep -E "Duration|Achieved Occupancy|Theoretical Occupancy|Registers Per|Block Limit|Warp Cycles Per Issued|Issue Slots Busy|DRAM Throughput|Memory Throughput|Waves Per SM|Grid Size" | cut -d, -f12-16
ncu -i gpurun_out/dec/attn.ncu-rep --page source --csv --print-source sass 2>/dev/null > gpurun_out/dec/attn_src.csv
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/dec/attn_src.csv')))
h=[r for r in rows if r and r[0]=='Address'][0]; si=h.index('Warp Stall Sampling (All Samples)')
body=[r for r in rows if r and r[0].startswith('0x')]
tot=sum(float(r[si] or 0) for r in body)
for r in sorted(body,key=lambda r:-float(r[si] or 0))[:15]: print(f"{float(r[si])/tot*100:5.1f}%", r[1][:90])
PY
