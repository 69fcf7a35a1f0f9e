#!/bin/bash
# compute-sanitizer over the step variants added late in round 1 (randomised
# step configurations, large beams, many bands, FAST tensor-core overlap).
mkdir -p gpurun_out/san2
export PYTHONFAULTHANDLER=1
K='fuzz or tensor_cores or step_matches_oracle'
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q --timeout 1400 -k "$K" -p no:cacheprovider > gpurun_out/san2/memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san2/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q --timeout 1400 -k "fuzz and (0 or 5 or 13 or 22 or 31)" -p no:cacheprovider > gpurun_out/san2/racecheck.log 2>&1; echo "exit $?" >> gpurun_out/san2/racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q --timeout 1100 -k "fuzz" -p no:cacheprovider > gpurun_out/san2/synccheck.log 2>&1; echo "exit $?" >> gpurun_out/san2/synccheck.log
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q --timeout 1100 -k "fuzz or tensor_cores" -p no:cacheprovider > gpurun_out/san2/initcheck.log 2>&1; echo "exit $?" >> gpurun_out/san2/initcheck.log
