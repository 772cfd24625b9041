mkdir -p gpurun_out/dec
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for G in 1 2; do
TIDAL_DEC_G=$G timeout 600 ncu --set full --import-source on --clock-control none -k regex:dec_gemv_bulk_kernel -s 41 -c 2 -o gpurun_out/dec/bulk_G$G -f python tools/decode_prof.py --steps 2 > gpurun_out/dec/ncu_full.log 2>&1
ncu -i gpurun_out/dec/bulk_G$G.ncu-rep --page details --csv 2>/dev/null | grep -E "Duration|Warp Cycles Per Issued|Issue Slots Busy|Stall|Memory Throughput|DRAM Throughput|Achieved Occupancy|Registers" | head -30
ncu -i gpurun_out/dec/bulk_G$G.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/dec/bulk_G$G.csv
done
