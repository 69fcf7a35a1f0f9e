#!/bin/bash
# ncu --set full captures of the full-vocabulary step's kernels at S=1 and S=64.
OUT=gpurun_out/${1:-ncu_full}
mkdir -p $OUT
for S in 1 64; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${2:-k_seg|k_logits}" -s 8 -c 6 \
    -f -o $OUT/full_s$S python scripts/full_probe.py $S 12 parity 3 > $OUT/log_s$S 2>&1
done
