#!/bin/bash
# Pair-row FP64 latency kernel (LANN_FP64_PRODUCERS=42) against the default: config-2 pass
# times, then its parity tests.
mkdir -p gpurun_out
out=gpurun_out/pair.txt
: > $out
for v in ${PVARS:-4 42 4 42}; do
  echo "== LANN_FP64_PRODUCERS=$v" >> $out
  LANN_FP64_PRODUCERS=$v timeout 300 python tools/prof_pop.py fp64 >> $out 2>&1
done
LANN_FP64_PRODUCERS=${PTEST:-42} timeout 1200 python -m pytest tests/test_gpu_full_length.py tests/test_gpu_parity.py tests/test_gpu_api.py -q -x 2>&1 | tail -8 > gpurun_out/pair_pytest.txt
cat $out gpurun_out/pair_pytest.txt
