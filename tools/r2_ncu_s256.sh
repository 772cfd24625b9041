# ncu --set full of the S = 256 GEMMs (cg 2, row-major weights), one launch each
O=gpurun_out/ncu256; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for n in qkv gate_up o down; do
  GB_ONLY=$n:2:0 timeout 300 ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 3 -c 1 -o $O/$n -f python tools/gemm_bench.py --S 256 --layout-ab --reps 2 > $O/$n.log 2>&1
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/$n.csv 2>/dev/null
done
python - <<'PY'
import csv
keys=['gpu__time_duration.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum',
'lts__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','lts__t_bytes.sum',
'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__cycles_active.avg','gpc__cycles_elapsed.max',
'l1tex__m_xbar2l1tex_read_bytes.sum','lts__d_sectors_fill_sysmem.sum','lts__t_sectors_srcunit_tex_op_read.sum',
'smsp__cycles_active.avg','sm__throughput.avg.pct_of_peak_sustained_elapsed','gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed']
for n in ['qkv','gate_up','o','down']:
    try: r=list(csv.reader(open(f'gpurun_out/ncu256/{n}.csv')))
    except Exception as e: print(n,e); continue
    h,u=r[0],r[1]
    for row in r[2:]:
        print(n)
        for k in keys:
            if k in h: print('   ',k,row[h.index(k)],u[h.index(k)])
        for i,k in enumerate(h):
            if ('lts__' in k or 'dram__' in k) and 'pct' in k and k not in keys: print('   ',k,row[i])
PY
