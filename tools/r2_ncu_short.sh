mkdir -p gpurun_out/short
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
TIDAL_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemm_tc_kernel<.int.(1|2|3), .int.(256|128|192), .int.2" -s 12 -c 4 -o gpurun_out/short/s256 -f python tools/warm.py --seq 256 --steps 1 --warmup 1 > gpurun_out/short/ncu256.log 2>&1
python tools/ncu_summary.py gpurun_out/short/s256.ncu-rep
ncu -i gpurun_out/short/s256.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keys=['Kernel Name','gpu__time_duration.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','l1tex__m_xbar2l1tex_read_bytes.sum','lts__t_bytes.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','lts__throughput.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum']
idx=[h.index(k) for k in keys if k in h]
for row in r[2:]:
    print([ (h[i].split('.')[0][-30:], row[i][:40]) for i in idx])
"
