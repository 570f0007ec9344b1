#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stfas.py tests/test_gpu_ops.py -x -q -k "shapes_agree or stencil or operator or sweep or vcycle" > gpurun_out/r02d_pytest.log 2>&1; echo pytest=$? >> gpurun_out/r02d_pytest.log
tail -3 gpurun_out/r02d_pytest.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg5 or cfg4" > gpurun_out/r02d_cfg.log 2>&1; echo pytest=$? >> gpurun_out/r02d_cfg.log
tail -3 gpurun_out/r02d_cfg.log
bash tools/gpu_rowtile.sh r02d
