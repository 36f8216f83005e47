#!/bin/bash
# Round-2 ncu captures of the FP32 kernels: the config-2 blur CTA kernel, the sweep's 5-5 warp
# kernel and the generic (unconstrained-shape) CTA kernel. Outputs -> gpurun_out/summary_*.txt
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k "regex:cta_kernel<\(int\)6, \(int\)5" -c 1 -o gpurun_out/prof_cta -f \
  python tools/prof_pop.py fp32 0 0.25 > gpurun_out/ncu_cta.log 2>&1
timeout 900 $NCU -k "regex:h55_kernel<\(int\)6" -c 1 -o gpurun_out/prof_h55 -f \
  python tools/sweep_parts.py 256 > gpurun_out/ncu_h55.log 2>&1
timeout 900 $NCU -k "regex:fp32_wide" -c 1 -o gpurun_out/prof_wide -f \
  python tools/unconstrained_probe.py > gpurun_out/ncu_wide.log 2>&1
for r in cta h55 wide; do
  [ -f gpurun_out/prof_$r.ncu-rep ] && python tools/ncu_summary.py gpurun_out/prof_$r.ncu-rep > gpurun_out/summary_$r.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/summary_cta.txt gpurun_out/summary_h55.txt gpurun_out/summary_wide.txt
