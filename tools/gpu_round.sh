#!/bin/bash
# One GPU session: parity tests, bench (+ reference arm), launch list, ncu captures.
# Outputs -> gpurun_out/ ; the summaries worth keeping are copied to profiles/ by hand.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch.err
if [ "${PROFILE:-1}" = "1" ]; then
  # config-2 CTA kernel (blur, the critical path) and the config-3 warp kernel (sweep)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"train_fp32_cta_kernel<6" -c 1 \
    -o gpurun_out/prof_cta -f python tools/prof_pop.py fp32 128 0.25 > gpurun_out/ncu_cta.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"train_fp32_kernel<7, 8, 0" -c 1 \
    -o gpurun_out/prof_warp -f python tools/prof_sweep.py 256 > gpurun_out/ncu_warp.log 2>&1
  python tools/prof_sweep.py 256 > gpurun_out/sweep.txt 2>&1
fi
tail -5 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; cat gpurun_out/bench_ref.json; cat gpurun_out/sweep.txt
