#!/bin/bash
# Short GPU iteration on the FP64 exact trainer: parity tests, phase profile, config-2 pass times.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_full_length.py tests/test_gpu_parity.py tests/test_gpu_api.py -q -x 2>&1 | tail -15 > gpurun_out/iter_pytest.txt
for v in "X=1" ${EXTRA_VARIANTS}; do
  echo "== $v" >> gpurun_out/iter_phase.txt
  env $v LANN_PHASE_PROFILE=1 timeout 300 python tools/prof_pop.py fp64 >> gpurun_out/iter_phase.txt 2>&1
  env $v timeout 300 python tools/prof_pop.py fp64 >> gpurun_out/iter_phase.txt 2>&1
done
cat gpurun_out/iter_pytest.txt gpurun_out/iter_phase.txt
