#!/bin/bash
# K4 iteration: parity tests of the step / config shapes / stages, then
# per-stage times for the new kernel (default) and the previous one
# (LSB_K4_LN=0) over batch sizes, then a short bench.
OUT=gpurun_out/${1:-k4}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_configs.py tests/test_gpu_stages.py -x -q --timeout 300 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for S in 1 16 64 128; do
  timeout 300 python scripts/stage_probe.py $S 12 >> $OUT/probe_new.txt 2>&1
  LSB_K4_LN=0 timeout 300 python scripts/stage_probe.py $S 12 >> $OUT/probe_old.txt 2>&1
done
timeout 300 python scripts/stage_probe.py 256 50 >> $OUT/probe_new.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 300 > $OUT/bench.json 2>$OUT/bench.err
