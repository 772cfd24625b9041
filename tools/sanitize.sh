# compute-sanitizer over the tiny / hd-128 workload; logs -> gpurun_out/sanitizer_<tool>[_fused].txt
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for f in 0 1; do
for tool in memcheck racecheck synccheck; do
  TIDAL_FUSED_SHRINK=$f timeout 1200 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_run.py > gpurun_out/sanitizer_${tool}_f$f.txt 2>&1
  echo "$tool fused=$f rc=$?"; tail -3 gpurun_out/sanitizer_${tool}_f$f.txt
done
done
