#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, ncu launch list and one
# `ncu --set full` capture of the named kernels. Outputs go to gpurun_out/.
# usage: scripts/gpu_round.sh [tag] [kernel-regex ...]
TAG=${1:-r01}
shift || true
KERNELS=${*:-k_logits k_probe_count k_compact k_softmax_topb k_expand}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > "$OUT/gpu.txt" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > "$OUT/pytest_gpu.log" 2>&1
echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke exit $?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" >> "$OUT/bench.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
  --no-extras > "$OUT/ncu_launch_bench.log" 2>&1
for k in $KERNELS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 60 -c 1 \
    -f -o "$OUT/prof_$k" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras \
    > "$OUT/ncu_full_$k.log" 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_tc_logits" -s 5 -c 1 \
  -f -o "$OUT/prof_k_tc_logits" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras \
  --mode fast > "$OUT/ncu_full_k_tc_logits.log" 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 200 --csv \
  --log-file "$OUT/launches_fast.csv" python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
  --no-extras --mode fast > "$OUT/ncu_launch_bench_fast.log" 2>&1
# the full-vocabulary path (the >= 4x denominator) at S=64: lane-kernel
# logits and the segmented softmax
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_logits_ln|^k_seg_" -s 4 -c 4 \
  -f -o "$OUT/prof_full_vocab" python scripts/full_probe.py 64 12 parity 2 > "$OUT/ncu_full_vocab.log" 2>&1
echo done > "$OUT/DONE"
