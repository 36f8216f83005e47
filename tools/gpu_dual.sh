#!/bin/bash
# FP64 pipelined trainer: single-round dual-sample producers (LANN_FP64_PRODUCERS=40) vs default
mkdir -p gpurun_out; rm -f gpurun_out/dual.txt
for n in ${NS:-4 40}; do
  echo "== producers $n" >> gpurun_out/dual.txt
  LANN_FP64_PRODUCERS=$n timeout 300 python tools/prof_pop.py fp64 >> gpurun_out/dual.txt 2>&1
  LANN_FP64_PRODUCERS=$n LANN_PHASE_PROFILE=1 timeout 300 python tools/prof_pop.py fp64 0 0.1 2>&1 | grep "6-5-5\|7-8-0" | head -2 >> gpurun_out/dual.txt
done
LANN_FP64_PRODUCERS=${PT:-40} timeout 900 python -m pytest tests/test_gpu_full_length.py tests/test_gpu_parity.py tests/test_cv.py -m gpu -q -x -k "fp64 or parity or exact or cv" 2>&1 | tail -3 >> gpurun_out/dual.txt
cat gpurun_out/dual.txt
