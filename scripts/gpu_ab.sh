#!/bin/bash
# Parity tests under ENV_B, then an interleaved bench A/B of the default
# build vs ENV_B (e.g. ENV_B="LSB_K4_EARLY=0"). usage: scripts/gpu_ab.sh TAG "ENV_B"
OUT=gpurun_out/${1:-ab}
ENVB=${2:-}
mkdir -p $OUT
env $ENVB timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_configs.py -x -q > $OUT/pytest_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_configs.py -x -q > $OUT/pytest_a.log 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 300 >> $OUT/bench_a.jsonl 2>>$OUT/bench.err
  env $ENVB timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 300 >> $OUT/bench_b.jsonl 2>>$OUT/bench.err
done
for S in 16 64 128; do
  timeout 300 python scripts/stage_probe.py $S 12 | grep lsh >> $OUT/probe_a.txt 2>&1
  env $ENVB timeout 300 python scripts/stage_probe.py $S 12 | grep lsh >> $OUT/probe_b.txt 2>&1
done
