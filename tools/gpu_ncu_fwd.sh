#!/bin/bash
# ncu --set full of the level-0 forward (first launch) and backward; raw pages exported to csv
TAG=${1:-r02t}
mkdir -p gpurun_out
CMD="python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-tts"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
for K in k_scgs_fwd k_scgs_back; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$K -c 1 \
      -o gpurun_out/${TAG}_$K $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_${K}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page details --csv > gpurun_out/${TAG}_${K}_details.csv 2>/dev/null
  rm -f gpurun_out/${TAG}_$K.ncu-rep
done
ls -la gpurun_out
