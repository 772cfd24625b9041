# full GPU suite + bench (one round-2 iteration)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1
tail -8 gpurun_out/gputests.log
timeout 900 python bench.py --steps 20 --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 300 gpurun_out/bench.err
python tools/show_bench.py gpurun_out/bench.json 2>/dev/null | head -30
