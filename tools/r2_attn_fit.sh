# paired attention: time vs (S, H) to separate per-item overhead from per-tile-step time
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for H in 40 74 148; do timeout 300 python tools/attn_bench.py --S 512 1024 2048 4096 8192 --H $H --reps 10; done
