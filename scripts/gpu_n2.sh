mkdir -p gpurun_out/n2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 200 --csv --log-file gpurun_out/n2/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/n2/l.log 2>&1
bash scripts/gpu_ncu.sh n2 k_softmax_topb
bash scripts/gpu_ncu.sh n2 k_expand
