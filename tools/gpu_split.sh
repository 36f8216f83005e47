#!/bin/bash
# FP64 latency kernel: where in a round's last block the chain waits for the next round
# (LANN_ROUND_SPLIT sample pairs linked first; 16 = after the whole block, the round-2 layout).
mkdir -p gpurun_out
out=gpurun_out/split_phase.txt
: > $out
for v in ${SPLITS:-16 8 12 4}; do
  touch paper_2003_07497_b200/csrc/train_fp64_pipe.cu
  make -C paper_2003_07497_b200/csrc NVCC="/usr/local/cuda/bin/nvcc -DLANN_ROUND_SPLIT=$v" ../lib/libperfsage_b200.so > gpurun_out/split_build_$v.log 2>&1 || { echo "build $v failed" >> $out; continue; }
  echo "== LANN_ROUND_SPLIT=$v" >> $out
  LANN_PHASE_PROFILE=1 timeout 300 python tools/prof_pop.py fp64 2>&1 | grep -E "6-5-5|7-8-0|ms" >> $out
  for r in 1 2; do timeout 300 python tools/prof_pop.py fp64 >> $out 2>&1; done
done
cat $out
