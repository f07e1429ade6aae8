# Round-2 call 3: full GPU suite, C2 bench (drop-in e2e), 2048 dense GETRF trace, C3/C5 quick bench.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; tail -c 1500 gpurun_out/r2_bench_c2.json; tail -3 gpurun_out/r2_bench_c2.err
timeout 300 python scripts/micro_getrf.py 2048 2048 5 --trace > gpurun_out/r2_getrf2048.txt 2>&1; cat gpurun_out/r2_getrf2048.txt | cut -c1-220
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_c3.json 2>/dev/null; python scripts/summarize.py < gpurun_out/r2_bench_c3.json | head -2
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_bench_c5.json 2>/dev/null; python scripts/summarize.py < gpurun_out/r2_bench_c5.json | head -2
