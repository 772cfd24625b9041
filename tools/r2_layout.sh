# NOTE: measured with an experimental patch that was not kept (see DESIGN.md 7d and
# profiles/short_r02.txt); the flags it uses no longer exist in the tree.
# row-major vs K-block-major weight boxes (DRAM locality), 13B GEMMs at S = 256 / 867 / 2048
mkdir -p gpurun_out/layout
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for S in 256 867 2048; do
  timeout 600 python tools/gemm_bench.py --S $S --layout-ab --reps 10 > gpurun_out/layout/S$S.txt 2>&1; echo S=$S; cat gpurun_out/layout/S$S.txt
done
