#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/diag_shape_oracle.py > gpurun_out/r02f_diag.log 2>&1; echo diag=$? >> gpurun_out/r02f_diag.log
cat gpurun_out/r02f_diag.log
timeout 600 python -m pytest tests/test_gpu_stfas.py -q -x -k "shapes_agree" > gpurun_out/r02f_pytest.log 2>&1; echo pytest=$? >> gpurun_out/r02f_pytest.log
tail -2 gpurun_out/r02f_pytest.log
Q="python bench.py --config 5 --steps 5 --warmup 3 --no-cpu --no-e2e --no-tts"
summ() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2], round(d['ms_per_step'],2), 'ms', {k:v['ms_per_step_by_level'] for k,v in d['kernels'].items()})" $1 "$2"; }
for V in bm2 bm3; do
  SMK_LIB_VARIANT=$V timeout 600 $Q > gpurun_out/r02f_$V.json 2> gpurun_out/r02f_$V.err; summ gpurun_out/r02f_$V.json $V
done
timeout 600 $Q > gpurun_out/r02f_base.json 2> gpurun_out/r02f_base.err; summ gpurun_out/r02f_base.json base
SMK_FWD_THRESH=200000,9472 timeout 600 $Q > gpurun_out/r02f_l1p2.json 2> gpurun_out/r02f_l1p2.err; summ gpurun_out/r02f_l1p2.json l1-tm32p2
CMD="python bench.py --config 5 --steps 1 --warmup 1 --no-cpu --no-e2e --no-tts"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_scgs_back -c 1 \
    -o gpurun_out/r02f_back $CMD > gpurun_out/r02f_ncu_back.log 2>&1
echo ncu=$?
