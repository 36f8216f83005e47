#!/bin/bash
# A/B of environment-selected kernel variants on the config-3 sweep parts and config 2.
# usage: VARIANTS="A=1 A=0" bash tools/gpu_ab.sh
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for v in $VARIANTS; do
  echo "== $v" >> gpurun_out/ab.txt
  env $v python tools/sweep_parts.py 256 >> gpurun_out/ab.txt 2>&1
  env $v python tools/prof_pop.py fp32 >> gpurun_out/ab.txt 2>&1
done
env $TESTENV python -m pytest tests/test_gpu_fp32.py -q -x 2>&1 | tail -3 >> gpurun_out/ab.txt
cat gpurun_out/ab.txt
