#!/bin/bash
# ncu --set full capture of one kernel inside a short bench run.
# usage: scripts/gpu_ncu.sh <tag> <kernel-regex> [bench args...]
TAG=$1; K=$2; shift 2
mkdir -p gpurun_out/$TAG
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 60 -c 1 \
  -f -o gpurun_out/$TAG/prof_$K python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras "$@" \
  > gpurun_out/$TAG/ncu_$K.log 2>&1
echo "exit $?" >> gpurun_out/$TAG/ncu_$K.log
