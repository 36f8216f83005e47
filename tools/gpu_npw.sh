#!/bin/bash
# FP64 pipelined trainer: producer-warp count sweep on config 2 (device ms per pass + phase split)
mkdir -p gpurun_out
for n in 4 5 6 8; do
  echo "== producers $n" >> gpurun_out/npw.txt
  LANN_FP64_PRODUCERS=$n timeout 300 python tools/prof_pop.py fp64 >> gpurun_out/npw.txt 2>&1
  LANN_FP64_PRODUCERS=$n LANN_PHASE_PROFILE=1 timeout 300 python tools/prof_pop.py fp64 0 0.1 2>&1 | grep "6-5-5\|7-8-0" | head -2 >> gpurun_out/npw.txt
done
cat gpurun_out/npw.txt
