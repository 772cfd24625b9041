# packed FFMA2 in the decode GEMV dot products: parity + same-box A/B against HEAD (ab/old)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_kernels.py -q -x -k "decode or attention or gemv" 2>&1 | tail -1
for r in 1 2 3; do
  timeout 300 python tools/decode_prof.py --steps 64 2>&1 | tail -1 | sed "s/^/new /"
  (cd ab/old && timeout 300 python tools/decode_prof.py --steps 64 2>&1 | tail -1 | sed "s/^/old /")
done
