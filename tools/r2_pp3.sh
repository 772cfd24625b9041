# LPT item schedule for the paired attention: parity + A/B (TIDAL_ATTN_LPT=0) + CTA end spread
mkdir -p gpurun_out/pp
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for r in 1 2; do for v in 1 0; do TIDAL_ATTN_LPT=$v timeout 300 python tools/attn_bench.py --S 867 1154 2048 4096 8192 --reps 10 | sed "s/^/lpt$v /"; done; done
for v in 1 0; do
TIDAL_ATTN_LPT=$v TIDAL_ATTN=2 TIDAL_ATTN_TRACE=gpurun_out/pp/t2048_$v.bin timeout 300 python tools/attn_bench.py --S 2048 --reps 1 > /dev/null
echo "lpt=$v"; python tools/attn_pp_trace.py gpurun_out/pp/t2048_$v.bin 2048 40 | tail -1
done
