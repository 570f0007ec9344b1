#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02j_ref.json 2> gpurun_out/r02j_ref.err; echo ref=$?
for C in 1 2 3 4; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-e2e > gpurun_out/r02j_c$C.json 2> gpurun_out/r02j_c$C.err; echo c$C=$?
done
timeout 900 python bench.py --config 4 --dtype fp64 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02j_c4f64.json 2> gpurun_out/r02j_c4f64.err; echo c4f64=$?
timeout 900 python bench.py --config 5 --dtype fp64 --steps 3 --warmup 3 --no-e2e --no-cpu --tts-budget 30 > gpurun_out/r02j_c5f64.json 2> gpurun_out/r02j_c5f64.err; echo c5f64=$?
timeout 1500 bash tools/profile_round.sh r02j 5
echo prof=$?
