#!/bin/bash
# compute-sanitizer passes over the GPU parity tests (memcheck, racecheck, synccheck, initcheck).
mkdir -p gpurun_out/san
export PYTHONFAULTHANDLER=1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_vocab_shard.py tests/test_gpu_step.py -x -q --timeout 900 -p no:cacheprovider > gpurun_out/san/memcheck.log 2>&1; echo "exit $?" >> gpurun_out/san/memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_vocab_shard.py -x -q --timeout 900 -k "3000 and 2" -p no:cacheprovider > gpurun_out/san/racecheck.log 2>&1; echo "exit $?" >> gpurun_out/san/racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q --timeout 800 -k "4000" -p no:cacheprovider > gpurun_out/san/synccheck.log 2>&1; echo "exit $?" >> gpurun_out/san/synccheck.log
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q --timeout 800 -k "4000" -p no:cacheprovider > gpurun_out/san/initcheck.log 2>&1; echo "exit $?" >> gpurun_out/san/initcheck.log
for i in $(seq 1 15); do timeout 200 python -m pytest tests/test_gpu_vocab_shard.py -x -q --timeout 150 -p no:cacheprovider > gpurun_out/san/stress_$i.log 2>&1 || echo "stress $i failed" >> gpurun_out/san/stress_fail.log; done
