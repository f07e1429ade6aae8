# Round-2 first box call: host probe, GPU suite, C2 bench, reference ladder on the box's host cores.
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv) > gpurun_out/r2_host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r2_bench_c2_start.json 2> gpurun_out/r2_bench_c2_start.err; tail -c 600 gpurun_out/r2_bench_c2_start.json
timeout 1500 python scripts/ref_ladder.py C2 16 24 32 40 48 --out gpurun_out/r2_ref_ladder_c2.jsonl 2>&1 | cut -c1-400
