mkdir -p gpurun_out/n4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' -c 200 --csv --log-file gpurun_out/n4/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras --mode fast > gpurun_out/n4/l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_logits' -s 5 -c 1 -f -o gpurun_out/n4/prof_k_tc_logits python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --mode fast > gpurun_out/n4/ncu_tc.log 2>&1
