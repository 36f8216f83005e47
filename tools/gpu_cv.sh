#!/bin/bash
# Round-2 session: cross-validation summary tests, the config-3 FP32 vs FP64-exact parity run, bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cv.py tests/test_gpu_cli.py tests/test_gpu_multi.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_cv.txt
timeout 1200 python tools/cv_parity.py ${SEEDS:-256} > gpurun_out/cv_parity.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/pytest_cv.txt; cat gpurun_out/cv_parity.log | head -60; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(json.dumps(d['extras']['config3_sweep_fp32'])[:3000])"
