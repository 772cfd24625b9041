mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_tp_wide.py tests/test_gpu_tp_local.py -q -m gpu -x > gpurun_out/tp_tests.log 2>&1
tail -15 gpurun_out/tp_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --quick --no-cpu-baseline > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
echo "torchrun rc=$?"; tail -c 400 gpurun_out/bench_torchrun1.err
python bench.py --gpus 2 --steps 1 ; echo "gpus2 rc=$?"
