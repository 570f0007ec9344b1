#!/bin/bash
# Profiling pass for the round's evidence (run under gpurun on ONE GPU):
#   1. plain bench (cfg given) -> gpurun_out/<tag>_bench.json
#   2. ncu launch list of one timed V-cycle (time + DRAM bytes per launch)
#   3. ncu --set full of the top kernel's first level-0 launch
# Each ncu run follows the identical command having exited 0 without ncu.
set -e
TAG=${1:-r01}
CFG=${2:-5}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu --no-e2e --no-tts"
mkdir -p gpurun_out
python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu > gpurun_out/${TAG}_c${CFG}_bench.json 2> gpurun_out/${TAG}_c${CFG}_bench.err
$CMD > gpurun_out/${TAG}_c${CFG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off -c 2000 --csv --log-file gpurun_out/${TAG}_c${CFG}_launches.csv $CMD \
    > gpurun_out/${TAG}_c${CFG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"${3:-k_scgs_fwd}" -c 1 \
    -o gpurun_out/${TAG}_c${CFG}_top $CMD > gpurun_out/${TAG}_c${CFG}_ncu_full.log 2>&1
