#!/bin/bash
# One GPU session: parity tests, bench, reference arm, launch list. Outputs -> gpurun_out/
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch.err
cat gpurun_out/pytest_gpu.txt | tail -15; cat gpurun_out/bench.json; cat gpurun_out/bench_ref.json
