#!/bin/bash
# compute-sanitizer over every colour-pass kernel shape (tools/sanitize_shapes.py)
mkdir -p gpurun_out
export SMK_NO_GRAPH=1
python tools/sanitize_shapes.py > gpurun_out/r02h_san_plain.log 2>&1; echo plain=$?
for T in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_shapes.py > gpurun_out/r02h_san_$T.log 2>&1
  echo "$T rc=$?"; tail -2 gpurun_out/r02h_san_$T.log
done
