#!/bin/bash
# one-chain-warp FP64 trainer (LANN_FP64_PRODUCERS=1) vs the default: timing, phases, parity
mkdir -p gpurun_out
for n in 4 1; do
  echo "== producers $n" >> gpurun_out/chain1.txt
  LANN_FP64_PRODUCERS=$n timeout 300 python tools/prof_pop.py fp64 >> gpurun_out/chain1.txt 2>&1
  LANN_FP64_PRODUCERS=$n LANN_PHASE_PROFILE=1 timeout 300 python tools/prof_pop.py fp64 0 0.1 2>&1 | grep "6-5-5\|7-8-0" | head -2 >> gpurun_out/chain1.txt
done
LANN_FP64_PRODUCERS=1 timeout 900 python -m pytest tests/test_gpu_full_length.py tests/test_gpu_parity.py tests/test_cv.py -m gpu -q -x -k "fp64 or parity or exact or cv" 2>&1 | tail -5 >> gpurun_out/chain1.txt
cat gpurun_out/chain1.txt
