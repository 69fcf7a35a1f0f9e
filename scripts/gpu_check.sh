set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_1806_00588_b200 as p; c=p.Context(0); print('ctx ok', c.sm_count)"
timeout 900 python -m pytest tests/test_gpu_stages.py -x -q 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_step.py -x -q 2>&1 | tail -30
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 600 python bench.py --steps 100 --warmup 5 --cpu-seconds 5 2>&1 | tail -5
