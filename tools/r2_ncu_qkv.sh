mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for v in 0 1; do
TIDAL_FUSED_SHRINK=$v TIDAL_GRAPH=0 timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:gemm_tc_kernel<.int.(1|3), .int.256, .int.2" -s 40 -c 4 -o gpurun_out/qkv_fused$v -f python tools/warm.py --steps 1 --warmup 1 > gpurun_out/ncu_q$v.log 2>&1
python tools/ncu_summary.py gpurun_out/qkv_fused$v.ncu-rep 2>&1 | head -30
done
