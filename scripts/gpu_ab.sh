#!/bin/bash
# A/B: default vs ENV_B (set by the caller), interleaved, plus the parity tests.
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_stages.py tests/test_gpu_vocab_shard.py -x -q --timeout 200 > gpurun_out/ab/pytest.log 2>&1; echo "exit $?" >> gpurun_out/ab/pytest.log
for rep in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 300 > gpurun_out/ab/A_$rep.json 2>/dev/null
  env ${ENV_B:-NOTHING=1} timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 300 > gpurun_out/ab/B_$rep.json 2>/dev/null
done
