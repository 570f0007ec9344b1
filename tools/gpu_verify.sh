#!/bin/bash
# round verification pass: smoke, every GPU test, the bench line (cfg5, with
# CPU baseline + e2e + time to solution), the reference arm, per-config lines,
# and the profiling pass (launch list + ncu --set full of the level-0
# forward and backward, exported to csv on the box)
TAG=${1:-r02u}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$? | tee -a gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo ref=$?
for C in 1 2 3 4; do
  timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-e2e > gpurun_out/${TAG}_c$C.json 2> gpurun_out/${TAG}_c$C.err; echo c$C=$?
done
timeout 900 python bench.py --config 4 --dtype fp64 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_c4f64.json 2> gpurun_out/${TAG}_c4f64.err
timeout 900 python bench.py --config 5 --dtype fp64 --steps 3 --warmup 3 --no-e2e --no-cpu --tts-budget 30 > gpurun_out/${TAG}_c5f64.json 2> gpurun_out/${TAG}_c5f64.err
timeout 1500 bash tools/profile_round.sh $TAG 5
CMD="python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-tts"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_scgs_back -c 1 \
    -o gpurun_out/${TAG}_back $CMD > gpurun_out/${TAG}_ncu_back.log 2>&1
for R in ${TAG}_c5_top ${TAG}_back; do
  ncu -i gpurun_out/$R.ncu-rep --page raw --csv > gpurun_out/${R}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$R.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/${R}_src.csv.gz
  rm -f gpurun_out/$R.ncu-rep
done
echo done
