mkdir -p gpurun_out/k5
for m in 0 1 2; do LSB_K5=$m timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 200 > gpurun_out/k5/bench_$m.json 2>&1; done
LSB_K5=1 timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_refsuite.py -x -q --timeout 300 > gpurun_out/k5/pytest1.log 2>&1
LSB_K5=2 timeout 600 python -m pytest tests/test_gpu_step.py -x -q --timeout 300 > gpurun_out/k5/pytest2.log 2>&1
