timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/micro_getrf.py 2048 2048 3 --trace 2>&1 | grep "ms/step\|GETRF k=1\|GETRF k=2"
timeout 900 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --levels-out gpurun_out/c2_levels_v68.npz 2>/dev/null | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
