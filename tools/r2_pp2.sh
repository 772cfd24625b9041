# ping-pong attention: exp2 split between MUFU and FMA (TIDAL_ATTN_EMU), pipelined head GEMV
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for emu in 0 2 4; do TIDAL_ATTN_EMU=$emu timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "attention or head" -x 2>&1 | tail -1; done
for i in 1 2; do
  echo "single"; TIDAL_ATTN=1 timeout 300 python tools/attn_bench.py --S 867 2048 8192
  for emu in 0 2 3 4; do echo "pp emu=$emu"; TIDAL_ATTN_EMU=$emu timeout 300 python tools/attn_bench.py --S 867 2048 8192; done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:head_kernel python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "head_logits" 2>&1 | grep -E "head_kernel|duration|dram" | head -8
