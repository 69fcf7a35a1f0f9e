mkdir -p gpurun_out/tc
timeout 120 python scripts/tc_check.py > gpurun_out/tc/check.log 2>&1
