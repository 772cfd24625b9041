mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 ) > gpurun_out/gputests.log 2>&1
tail -25 gpurun_out/gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --quick --no-cpu-baseline --no-sweep > gpurun_out/ncu_launch.log 2>&1
python tools/launches.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1; cat gpurun_out/launches.txt
