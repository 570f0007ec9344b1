#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lbfgs.py -q -s > gpurun_out/r02o_lbfgs.log 2>&1; echo pytest=$? >> gpurun_out/r02o_lbfgs.log
grep -E "lbfgs\]|passed|failed|Error" gpurun_out/r02o_lbfgs.log | tail -12
python -m paper_1608_01102_b200.cli make-benchmark --name translated-blob --res 32 --frames 10 --out /tmp/tb > /dev/null
timeout 1200 python -m paper_1608_01102_b200.cli compare-baseline --config /tmp/tb/run.cfg --out gpurun_out/r02o_compare > gpurun_out/r02o_compare.log 2>&1; echo compare=$? >> gpurun_out/r02o_compare.log
cat gpurun_out/r02o_compare.log | tail -5
