mkdir -p gpurun_out/n5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_logits' -s 5 -c 1 -f -o gpurun_out/n5/prof_k_logits_fast python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --mode fast > gpurun_out/n5/a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tc_logits' -s 5 -c 1 -f -o gpurun_out/n5/prof_k_tc_logits python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --mode fast > gpurun_out/n5/b.log 2>&1
