mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputests.log 2>&1
tail -6 gpurun_out/gputests.log
bash tools/r2_ab_warm.sh
