#!/bin/bash
# compute-sanitizer over the round-2 kernels: k_logits_ln (full vocabulary and
# forced onto the LSH step), k_seg_* (segmented softmax), k_probe_split (few
# rows x many bands), CUDA-graph replay, the packed vocabulary-sharded step,
# the shared-memory cuckoo build.
OUT=gpurun_out/san2
mkdir -p $OUT
export PYTHONFAULTHANDLER=1
SEL="full_vocab or graph or 9000 or 12000 or 1500-256 or 2000-64-8-3-100"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q -k "$SEL" -p no:cacheprovider > $OUT/memcheck.log 2>&1; echo "exit $?" >> $OUT/memcheck.log
LSB_K4_LN=2 timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q -k "test_step_matches_oracle and 4000" -p no:cacheprovider > $OUT/memcheck_ln2.log 2>&1; echo "exit $?" >> $OUT/memcheck_ln2.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q -k "full_vocab and 9000 or 1500-256" -p no:cacheprovider > $OUT/racecheck.log 2>&1; echo "exit $?" >> $OUT/racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q -k "full_vocab and 9000 or 1500-256" -p no:cacheprovider > $OUT/synccheck.log 2>&1; echo "exit $?" >> $OUT/synccheck.log
timeout 1500 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q -k "full_vocab and 9000 or 1500-256" -p no:cacheprovider > $OUT/initcheck.log 2>&1; echo "exit $?" >> $OUT/initcheck.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_vocab_shard.py tests/test_gpu_dropin.py -x -q -k "not wtaidx" -p no:cacheprovider > $OUT/memcheck_shard_dropin.log 2>&1; echo "exit $?" >> $OUT/memcheck_shard_dropin.log
for i in $(seq 1 10); do timeout 300 python -m pytest tests/test_gpu_step.py -x -q -k "graph or full_vocab or 12000" -p no:cacheprovider > $OUT/stress_$i.log 2>&1 || echo "stress $i failed" >> $OUT/stress_fail.log; done
