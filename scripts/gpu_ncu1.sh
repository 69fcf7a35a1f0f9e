#!/bin/bash
# One `ncu --set full` capture of the PARITY bench's k_logits (and optionally
# other kernels) into gpurun_out/ncu1/. usage: scripts/gpu_ncu1.sh [regex] [bench args]
K=${1:-k_logits}
shift || true
mkdir -p gpurun_out/ncu1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K" -s 60 -c 1 \
  -f -o gpurun_out/ncu1/prof python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras "$@" \
  > gpurun_out/ncu1/log 2>&1
echo "exit $?" >> gpurun_out/ncu1/log
