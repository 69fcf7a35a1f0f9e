#!/bin/bash
# Quick GPU check: parity suite (per-test timeout) + bench lines (parity, fast).
mkdir -p gpurun_out/q
timeout 120 python scripts/tc_check.py > gpurun_out/q/tc_check.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/q/pytest.log 2>&1; echo "exit $?" >> gpurun_out/q/pytest.log
timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/q/bench.json 2> gpurun_out/q/bench.err
timeout 200 python bench.py --no-cpu-baseline --no-extras --mode fast --steps 200 > gpurun_out/q/bench_fast.json 2>> gpurun_out/q/bench.err
