#!/bin/bash
# Round-2 GPU session: parity tests, bench (+ reference arm), launch list, ncu of the headline kernel.
# Outputs -> gpurun_out/ ; tools/ncu_summary.py turns the .ncu-rep files into profiles/ text.
mkdir -p gpurun_out
TESTS=${TESTS:-tests}
timeout 1500 python -m pytest $TESTS -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${REF:-1}" = "1" ]; then
  timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch.err
if [ "${PROFILE:-1}" = "1" ]; then
  NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
  # config-2 critical path in the FP64 exact headline: the pipelined blur-net trainer
  timeout 900 $NCU -k "regex:train_fp64_pipe<\(int\)6, \(int\)5" -c 1 -o gpurun_out/prof_fp64pipe -f \
    python tools/prof_pop.py fp64 0 0.1 > gpurun_out/ncu_fp64pipe.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_fp64pipe.ncu-rep > gpurun_out/summary_fp64pipe.txt 2>&1
  ncu -i gpurun_out/prof_fp64pipe.ncu-rep --page raw --csv > gpurun_out/raw_fp64pipe.csv 2>/dev/null
fi
LANN_PHASE_PROFILE=1 timeout 300 python tools/prof_pop.py fp64 > gpurun_out/phase_fp64.txt 2>&1
rm -f gpurun_out/*.ncu-rep
tail -5 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; cat gpurun_out/bench_ref.json 2>/dev/null; cat gpurun_out/phase_fp64.txt
