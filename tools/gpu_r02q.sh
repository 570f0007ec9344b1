#!/bin/bash
# profiling pass that exports csv summaries on the box and drops the (large) reports
mkdir -p gpurun_out
timeout 1500 bash tools/profile_round.sh r02q 5
CMD="python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-tts"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_scgs_back -c 1 \
    -o gpurun_out/r02q_back $CMD > gpurun_out/r02q_ncu_back.log 2>&1
for R in r02q_c5_top r02q_back; do
  ncu -i gpurun_out/$R.ncu-rep --page raw --csv > gpurun_out/${R}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$R.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${R}_src.csv 2>/dev/null
  gzip -f gpurun_out/${R}_src.csv
  rm -f gpurun_out/$R.ncu-rep
done
ls -la gpurun_out
