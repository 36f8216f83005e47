#!/bin/bash
# FP64 pipelined trainer: phase profile (contended / chain-after-production) + ncu source-level stalls
mkdir -p gpurun_out
for f in 0 1; do echo "== LANN_PROF_FLAGS=$f"; LANN_PROF_FLAGS=$f LANN_PHASE_PROFILE=1 python tools/prof_pop.py fp64 0 0.2 2>&1 | head -1; done > gpurun_out/prof_phase.txt
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:train_fp64_pipe<\(int\)6, \(int\)5" -c 1 -o gpurun_out/pipe -f python tools/prof_pop.py fp64 0 0.05 > gpurun_out/pipe.log 2>&1
ncu -i gpurun_out/pipe.ncu-rep --page source --csv --print-source sass > gpurun_out/pipe_sass.csv 2>&1
python tools/ncu_summary.py gpurun_out/pipe.ncu-rep > gpurun_out/pipe_summary.txt 2>&1
rm -f gpurun_out/pipe.ncu-rep
cat gpurun_out/prof_phase.txt gpurun_out/pipe_summary.txt
