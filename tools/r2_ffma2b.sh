# packed FFMA2 / FADD2 in the single-tile attention softmax (TIDAL_ATTN=1): parity + same-box A/B against HEAD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -1
for r in 1 2 3; do
  TIDAL_ATTN=1 timeout 300 python tools/attn_bench.py --S 867 2048 8192 --reps 10 | sed "s/^/new /"
  (cd ab/old && TIDAL_ATTN=1 timeout 300 python tools/attn_bench.py --S 867 2048 8192 --reps 10 | sed "s/^/old /")
done
