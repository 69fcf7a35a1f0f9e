#!/bin/bash
# One `ncu --set full` capture of one kernel of the PARITY bench into
# gpurun_out/<tag>/. usage: scripts/gpu_ncu1.sh <tag> <kernel regex> [bench args]
TAG=${1:-ncu1}; K=${2:-k_logits}
shift 2 || true
mkdir -p gpurun_out/$TAG
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 60 -c 1 \
  -f -o gpurun_out/$TAG/prof python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras "$@" \
  > gpurun_out/$TAG/log 2>&1
echo "exit $?" >> gpurun_out/$TAG/log
