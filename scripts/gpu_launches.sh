#!/bin/bash
# ncu launch list (per-kernel device time) of a short bench run; args go to bench.py
T=${TAG:-ll}
mkdir -p gpurun_out/$T
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 200 --csv --log-file gpurun_out/$T/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras "$@" > gpurun_out/$T/l.log 2>&1
