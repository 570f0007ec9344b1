#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_hygiene.py -q > gpurun_out/r02i_hygiene.log 2>&1; echo pytest=$? >> gpurun_out/r02i_hygiene.log
tail -15 gpurun_out/r02i_hygiene.log
