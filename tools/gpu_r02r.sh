#!/bin/bash
# verification pass on the current tree: smoke, GPU tests, bench (cfg5), launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r_smoke.log 2>&1; echo smoke=$? | tee -a gpurun_out/r02r_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02r_pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r02r_pytest_gpu.log
tail -15 gpurun_out/r02r_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/r02r_bench.json'));print(d['ms_per_step'], d['roofline']['frac'], {k:(v['vcycles_to_eps'],v['s_to_solution']) for k,v in d['time_to_solution'].items()})"
timeout 1200 bash tools/profile_round.sh r02r 5 > gpurun_out/r02r_profile.log 2>&1; echo profile=$?
ls gpurun_out
