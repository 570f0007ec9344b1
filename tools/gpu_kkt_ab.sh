#!/bin/bash
# k_kkt frames-per-thread check: per-config k_kkt / stop-test times, then every GPU test
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.load(open(sys.argv[1]));t=(d.get('time_to_solution') or {}).get('config_levels') or {};print(sys.argv[2], round(d['ms_per_step'],3), 'ms', d['kernels']['k_kkt']['ms_per_step_by_level'], 'stop test', t.get('stop_test_ms_per_cycle'), d['config']['residual_inf_after'])" $1 "$2"; }
for C in 5 4 3 2 1; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu --no-e2e --tts-budget 8 > gpurun_out/kkt_c$C.json 2> gpurun_out/kkt_c$C.err; summ gpurun_out/kkt_c$C.json "cfg$C"
done
timeout 300 python bench.py --config 4 --dtype fp64 --steps 3 --warmup 3 --no-cpu --no-e2e --tts-budget 8 > gpurun_out/kkt_c4f64.json 2>/dev/null; summ gpurun_out/kkt_c4f64.json c4f64
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02z_pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r02z_pytest_gpu.log; tail -4 gpurun_out/r02z_pytest_gpu.log
