timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --config C5 --steps 3 --warmup 2 --no-cpu --levels-out gpurun_out/c5_levels_v43.npz 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -4
timeout 1500 python scripts/balance_bench.py C5 --sizes 500,1000,2000,5000 --repeats 3 --out gpurun_out/balance_c5_v43.jsonl 2>&1 | grep "^#" | cut -c1-300
