#!/bin/bash
# One GPU session: parity tests, bench (+ reference arm), launch list, ncu captures.
# Outputs -> gpurun_out/ ; tools/ncu_summary.py turns the .ncu-rep files into profiles/ text.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-extras --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch.err
if [ "${PROFILE:-1}" = "1" ]; then
  NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
  # config-2 critical path: the blur CTA kernel
  timeout 900 $NCU -k "regex:cta_kernel<\(int\)6, \(int\)5" -c 1 -o gpurun_out/prof_cta -f \
    python tools/prof_pop.py fp32 0 0.25 > gpurun_out/ncu_cta.log 2>&1
  # config-3 sweep: the packed H=8 warp kernel and the blur warp kernel
  timeout 900 $NCU -k "regex:h8_kernel<\(int\)7" -c 1 -o gpurun_out/prof_h8 -f \
    python tools/sweep_parts.py 256 > gpurun_out/ncu_h8.log 2>&1
  # FP64 exact (parity mode) and the config-4 scorer
  timeout 600 $NCU -k "regex:exact<\(int\)1, \(int\)6" -c 1 -o gpurun_out/prof_fp64 -f \
    python tools/prof_pop.py fp64 0 0.1 > gpurun_out/ncu_fp64.log 2>&1
  timeout 600 $NCU -k "regex:select_variants_fast" --launch-skip 1 -c 1 -o gpurun_out/prof_select -f \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_select.log 2>&1
  python tools/sweep_parts.py 256 > gpurun_out/sweep.txt 2>&1
  python tools/prof_sweep.py 256 >> gpurun_out/sweep.txt 2>&1
fi
for r in cta h8 fp64 select; do
  [ -f gpurun_out/prof_$r.ncu-rep ] && python tools/ncu_summary.py gpurun_out/prof_$r.ncu-rep > gpurun_out/summary_$r.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep  # keep the copy-back under gpurun's size cap; summaries carry the numbers
tail -5 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; cat gpurun_out/bench_ref.json; cat gpurun_out/sweep.txt
