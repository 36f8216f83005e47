#!/bin/bash
# Short GPU iteration: FP32 tests, config-2 phase profile per CTA-kernel variant, bench.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fp32.py -q -x 2>&1 | tail -15 > gpurun_out/iter_pytest.txt
for v in "LANN_CTA_PAIR=1" "LANN_CTA_PAIR=0" "LANN_CTA_PACKED=1" ${EXTRA_VARIANTS}; do
  echo "== $v" >> gpurun_out/iter_phase.txt
  env $v LANN_PHASE_PROFILE=1 python tools/prof_pop.py fp32 >> gpurun_out/iter_phase.txt 2>&1
  env $v python tools/prof_pop.py fp32 >> gpurun_out/iter_phase.txt 2>&1
done
python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/iter_bench.json 2>&1
cat gpurun_out/iter_pytest.txt gpurun_out/iter_phase.txt gpurun_out/iter_bench.json
