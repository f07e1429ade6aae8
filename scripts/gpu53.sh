timeout 1500 python scripts/balance_bench.py C3 --sizes 2000,5000 --repeats 2 --out gpurun_out/r1_balance_c3.jsonl 2>&1 | grep "^#" | cut -c1-300
timeout 1500 python scripts/balance_bench.py C5 --repeats 3 --taus 0.05,0.1,0.25,0.5,off --out gpurun_out/r1_balance_c5.jsonl 2>&1 | grep "^#" | cut -c1-300
timeout 1500 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu --levels-out gpurun_out/c3_levels_v53.npz 2>&1 | tail -1 | python scripts/summarize.py 2>/dev/null | head -1
