# short-prompt breakdown: warm rho=1 per-kernel tables + ncu launch lists at S=256/867
mkdir -p gpurun_out/short
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for S in 256 867; do
  timeout 300 python tools/warm.py --seq $S --steps 10 --profile --tag S$S > gpurun_out/short/warm$S.json
  cat gpurun_out/short/warm$S.json
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/short/launches$S.csv python tools/warm.py --seq $S --steps 1 --warmup 1 > gpurun_out/short/ncu$S.log 2>&1
  python tools/launches.py gpurun_out/short/launches$S.csv > gpurun_out/short/launches$S.txt; head -30 gpurun_out/short/launches$S.txt
done
