# decode GEMV: residual rows split into K halves (default) vs row pairs (TIDAL_DEC_SPLIT=0); parity + timing + ncu list
mkdir -p gpurun_out/dec
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_decode.py -q -x > gpurun_out/dec/tests.log 2>&1; tail -3 gpurun_out/dec/tests.log
for v in 1 0 1 0; do
  TIDAL_DEC_SPLIT=$v timeout 300 python tools/decode_prof.py --steps 64 2>&1 | tail -1 | sed "s/^/split=$v /"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/dec/launches.csv python tools/decode_prof.py --steps 4 > gpurun_out/dec/ncu.log 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/dec/launches.csv')))
hi=[i for i,r in enumerate(rows) if "Kernel Name" in r][0]
h=rows[hi]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
agg=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[hi+1:]:
    if len(r)>vi: agg[r[ki].split("(")[0]][r[mi]].append(float(r[vi].replace(",","")))
for k,m in agg.items():
    if 'dec_' in k or 'head' in k:
        t=m['gpu__time_duration.sum']; b=m['dram__bytes_read.sum']; n=len(t)
        print(f"{k[:44]:44s} n={n:4d} mean {sum(t)/n/1e3:7.2f} us  {sum(b)/n/1e6:8.2f} MB  {sum(b)/sum(t):7.1f} GB/s")
PY
