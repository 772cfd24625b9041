# paired softmax: exponentials with the current reference computed before the row max (redo when
# the max grows > 2^8): parity + same-box A/B vs HEAD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -1
for r in 1 2 3; do
  timeout 300 python tools/attn_bench.py --S 1154 2048 4096 8192 --reps 10 | sed "s/^/new /"
  (cd ab/old && timeout 300 python tools/attn_bench.py --S 1154 2048 4096 8192 --reps 10 | sed "s/^/head /")
done
