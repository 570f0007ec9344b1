#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/diag_shape_oracle.py > gpurun_out/r02e_diag.log 2>&1; echo diag=$? >> gpurun_out/r02e_diag.log
cat gpurun_out/r02e_diag.log
timeout 900 python -m pytest tests/test_gpu_stfas.py tests/test_gpu_convergence.py tests/test_gpu_ops.py -q -k "singular or solve or converge or stencil or operator or residual" > gpurun_out/r02e_pytest.log 2>&1; echo pytest=$? >> gpurun_out/r02e_pytest.log
tail -5 gpurun_out/r02e_pytest.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg1 or cfg2" > gpurun_out/r02e_cfg.log 2>&1; echo pytest=$? >> gpurun_out/r02e_cfg.log
tail -3 gpurun_out/r02e_cfg.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
python -c "import json;d=json.load(open('gpurun_out/r02e_bench.json'));t=d['time_to_solution'];print(d['ms_per_step'], {k:(v['vcycles_to_eps'],v['s_to_solution'],v['stop_test_ms_per_cycle']) for k,v in t.items()})"
