# full GPU suite + sanitizer + bench (round-2 checkpoint)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1
tail -15 gpurun_out/gputests.log
cat gpurun_out/des_check.json 2>/dev/null
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 300 gpurun_out/bench.err
python tools/show_bench.py gpurun_out/bench.json 2>/dev/null | head -30
