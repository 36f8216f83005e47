#!/bin/bash
# FP64 latency kernel: round-0 producer stagger sweep (phase profile + config-2 pass time per
# setting), then the full-length parity tests with a stagger on.
mkdir -p gpurun_out
out=gpurun_out/stagger_phase.txt
: > $out
for v in ${STAGGERS:-0,0 200,0 300,0 400,0 500,0 300,150}; do
  echo "== LANN_FP64_STAGGER=$v" >> $out
  LANN_FP64_STAGGER=$v LANN_PHASE_PROFILE=1 timeout 300 python tools/prof_pop.py fp64 2>&1 | grep -E "6-5-5|7-8-0|ms" >> $out
  LANN_FP64_STAGGER=$v timeout 300 python tools/prof_pop.py fp64 >> $out 2>&1
done
LANN_FP64_STAGGER=${PARITY_STAGGER:-300,0} timeout 900 python -m pytest tests/test_gpu_full_length.py -q -x 2>&1 | tail -5 > gpurun_out/stagger_pytest.txt
cat $out gpurun_out/stagger_pytest.txt
