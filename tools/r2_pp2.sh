# cross-item S_A(0) in the paired attention: parity (variants 1/2/3) + A/B timing + trace
mkdir -p gpurun_out/pp
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_e2e.py -q -x -k "batch" 2>&1 | tail -2
for r in 1 2; do for v in 2 3; do TIDAL_ATTN=$v timeout 300 python tools/attn_bench.py --S 867 1154 2048 4096 8192 --reps 10 | sed "s/^/v$v /"; done; done
TIDAL_ATTN=2 TIDAL_ATTN_TRACE=gpurun_out/pp/t2048.bin timeout 300 python tools/attn_bench.py --S 2048 --reps 1 | tail -1
python tools/attn_pp_trace.py gpurun_out/pp/t2048.bin 2048 40
