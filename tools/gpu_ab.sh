#!/bin/bash
# A/B of libsmk variants on cfg5: bench V-cycle (per-kernel breakdown) for each
# variant name given ("base" = libsmk.so), alternating twice.
TAG=${TAG:-ab}
mkdir -p gpurun_out
Q="python bench.py --config ${CFG:-5} --steps 5 --warmup 3 --no-cpu --no-e2e --no-tts"
summ() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2], round(d['ms_per_step'],2), 'ms', {k:v['ms_per_step_by_level'] for k,v in d['kernels'].items() if k in ('k_scgs_fwd','k_scgs_back','k_kkt')})" $1 "$2"; }
for rep in 1 2; do
for V in "$@"; do
  if [ "$V" = base ]; then unset SMK_LIB_VARIANT; else export SMK_LIB_VARIANT=$V; fi
  timeout 600 $Q > gpurun_out/${TAG}_${V}_$rep.json 2> gpurun_out/${TAG}_${V}_$rep.err; summ gpurun_out/${TAG}_${V}_$rep.json "$V#$rep"
done
done
unset SMK_LIB_VARIANT
