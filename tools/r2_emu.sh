# FMA-pipe exp2 (packed) for 0..2 of every 4 groups of 8 P columns (TIDAL_ATTN_EMU): parity + A/B
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
TIDAL_ATTN_EMU=2 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -1
for r in 1 2 3; do for v in 0 1 2; do TIDAL_ATTN_EMU=$v timeout 300 python tools/attn_bench.py --S 2048 4096 8192 --reps 10 | sed "s/^/emu$v /"; done; done
