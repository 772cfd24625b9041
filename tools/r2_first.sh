mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r2_0.json 2> gpurun_out/bench_r2_0.err
tail -c 600 gpurun_out/bench_r2_0.err
python tools/show_bench.py gpurun_out/bench_r2_0.json 2>/dev/null | head -40
