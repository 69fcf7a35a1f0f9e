mkdir -p gpurun_out/n10
for k in k_softmax_topb k_expand k_compact; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 10 -c 1 -f -o gpurun_out/n10/prof_$k python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/n10/$k.log 2>&1
done
