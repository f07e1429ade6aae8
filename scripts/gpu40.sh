timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --levels-out gpurun_out/c2_levels_v40.npz 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -4
LBK_EXEC_PER_SM=1 timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
