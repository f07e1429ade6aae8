nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m "gpu" -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python bench.py --config C2 --steps 5 --warmup 3 --levels-out gpurun_out/c2_levels_v23.npz > gpurun_out/bench_c2_v23.json 2> gpurun_out/bench_c2_v23.log; tail -1 gpurun_out/bench_c2_v23.json | python scripts/summarize.py
