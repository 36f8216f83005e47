#!/bin/bash
# End-of-round GPU session: the round-2 session (tests, bench, reference arm, launch list, ncu of
# the headline kernel, phase profile) + smoke() + the N=2 bench path on one device (ranks share
# device 0: exercises the torchrun / gloo plumbing only).
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
bash tools/gpu_r02.sh
LANN_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-extras \
  > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err
cat gpurun_out/smoke.txt gpurun_out/bench_n2_shared.json
