set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r02c_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02c_pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r02c_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo bench=$?
tail -5 gpurun_out/r02c_pytest_gpu.log
