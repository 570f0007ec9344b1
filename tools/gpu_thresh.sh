#!/bin/bash
# hand-off format / forward shape thresholds at run time (no rebuild): cfg5 V-cycle per-level breakdown
Q="python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-tts"
summ() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2], round(d['ms_per_step'],2), 'ms', {k:v['ms_per_step_by_level'] for k,v in d['kernels'].items() if k in ('k_scgs_fwd','k_scgs_back')}, d['config']['residual_inf_after'])" $1 "$2"; }
$Q > gpurun_out/th_base.json 2> gpurun_out/th_base.err; summ gpurun_out/th_base.json base
SMK_CMP_MIN=100000000 $Q > gpurun_out/th_c.json 2> gpurun_out/th_c.err; summ gpurun_out/th_c.json "factored hand-off at level 0 (TM64/P2)"; tail -2 gpurun_out/th_c.err
$Q > gpurun_out/th_base2.json 2> gpurun_out/th_base2.err; summ gpurun_out/th_base2.json base
SMK_CMP_MIN=100000000 $Q > gpurun_out/th_c2.json 2> gpurun_out/th_c2.err; summ gpurun_out/th_c2.json "factored hand-off at level 0 (TM64/P2)"
