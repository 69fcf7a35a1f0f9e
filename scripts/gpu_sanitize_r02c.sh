#!/bin/bash
# compute-sanitizer over the round-2c additions: the single-launch cooperative
# step (LSB_FUSED=1), the glibc exp / log device functions, the certified
# softmax denominator and its sequential fallback (LSB_SEQ_DENOM=1), the
# multi-CTA K5b hidden reorder.
OUT=gpurun_out/san3
mkdir -p $OUT
export PYTHONFAULTHANDLER=1
SEL="fused_small or sequential_denominator or config1 or graph"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_step.py -x -q -k "$SEL" -p no:cacheprovider > $OUT/$tool.log 2>&1; echo "exit $?" >> $OUT/$tool.log
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_stages.py tests/test_gpu_glibc_log.py -x -q -k "softmax or log or exp" -p no:cacheprovider > $OUT/memcheck_softmax.log 2>&1; echo "exit $?" >> $OUT/memcheck_softmax.log
LSB_SEQ_DENOM=1 timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_stages.py -x -q -k "softmax_parity and False" -p no:cacheprovider > $OUT/racecheck_seq.log 2>&1; echo "exit $?" >> $OUT/racecheck_seq.log
echo done > $OUT/DONE
