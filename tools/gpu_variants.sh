#!/bin/bash
# FP64 latency kernel: compile-time variants of train_fp64_pipe.cu (VARIANTS = space-separated
# lists of -D flags joined by ','), phase profile + config-2 pass times each; then the default
# build's FP64 parity tests.
mkdir -p gpurun_out
out=gpurun_out/variants_phase.txt
: > $out
build() {
  touch paper_2003_07497_b200/csrc/train_fp64_pipe.cu
  make -C paper_2003_07497_b200/csrc NVCC="/usr/local/cuda/bin/nvcc $1" ../lib/libperfsage_b200.so > gpurun_out/variant_build.log 2>&1
}
for v in ${VARIANTS}; do
  flags=$(echo "$v" | tr ',' ' ')
  build "$flags" || { echo "build $v failed" >> $out; continue; }
  echo "== $v" >> $out
  LANN_PHASE_PROFILE=1 timeout 300 python tools/prof_pop.py fp64 2>&1 | grep -E "6-5-5|7-8-0|ms" >> $out
  for r in 1 2; do timeout 300 python tools/prof_pop.py fp64 >> $out 2>&1; done
done
build "" && timeout 1200 python -m pytest tests/test_gpu_full_length.py tests/test_gpu_parity.py tests/test_gpu_api.py -q -x 2>&1 | tail -5 > gpurun_out/variants_pytest.txt
cat $out gpurun_out/variants_pytest.txt
