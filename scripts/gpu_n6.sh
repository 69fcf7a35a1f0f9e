mkdir -p gpurun_out/n6
for k in k_probe_count k_compact k_softmax_topb k_expand; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 10 -c 1 -f -o gpurun_out/n6/prof_$k python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/n6/$k.log 2>&1
done
