#!/bin/bash
# final-tree pass: smoke, the default bench line, cfg3 / cfg4 lines, every GPU test
TAG=${1:-r02z}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$? | tee -a gpurun_out/${TAG}_smoke.log
summ() { python -c "import json,sys;d=json.load(open(sys.argv[1]));t=(d.get('time_to_solution') or {}).get('config_levels') or {};print(sys.argv[2], round(d['ms_per_step'],3), 'ms', d['kernels']['k_kkt']['ms_per_step_by_level'], 'stop test', t.get('stop_test_ms_per_cycle'), 'tts', {k:(v['vcycles_to_eps'], v['s_to_solution']) for k,v in (d.get('time_to_solution') or {}).items()})" $1 "$2"; }
timeout 700 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench=$?; summ gpurun_out/${TAG}_bench.json cfg5
for C in 4 3 2 1; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-e2e > gpurun_out/${TAG}_c$C.json 2> gpurun_out/${TAG}_c$C.err; summ gpurun_out/${TAG}_c$C.json "cfg$C"
done
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/${TAG}_pytest_gpu.log; tail -3 gpurun_out/${TAG}_pytest_gpu.log
