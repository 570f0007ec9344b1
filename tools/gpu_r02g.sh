#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_stfas.py -q -x -k "slab or shapes_agree or singular" > gpurun_out/r02g_pytest.log 2>&1; echo pytest=$? >> gpurun_out/r02g_pytest.log
tail -3 gpurun_out/r02g_pytest.log
timeout 1500 python tools/slab_convergence.py --config 5 --slabs 1 2 4 8 --levels 0 99 --budget 80 > gpurun_out/r02g_slabconv.jsonl 2> gpurun_out/r02g_slabconv.err; echo conv=$?
python -c "
import json
for l in open('gpurun_out/r02g_slabconv.jsonl'):
    d=json.loads(l); print(d['slabs'], d['levels'], d['vcycles_to_eps'], round(d['asym_factor'] or 0,3), round(d['ms_per_vcycle_serialised'],1))
"
tail -3 gpurun_out/r02g_slabconv.err
