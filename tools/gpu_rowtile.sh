#!/bin/bash
# Row-order experiment (color_cell banded rows): bench cfg5 V-cycle at
# SMK_ROW_TILE = 1 (plain), 4, 8, 16; then the profiling pass at the default.
TAG=${1:-r02c}
mkdir -p gpurun_out
Q="python bench.py --config 5 --steps 5 --warmup 3 --no-cpu --no-e2e --no-tts"
for T in 1 4 8 16; do
  SMK_ROW_TILE=$T timeout 600 $Q > gpurun_out/${TAG}_rt${T}.json 2> gpurun_out/${TAG}_rt${T}.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_rt${T}.json'));print('T=$T', round(d['ms_per_step'],2), 'ms', {k:v['ms_per_step_by_level'] for k,v in d['kernels'].items()})"
done
timeout 1200 bash tools/profile_round.sh $TAG 5
python tools/launch_summary.py gpurun_out/${TAG}_c5_launches.csv 2>&1 | tail -3
