( while true; do free -g | awk 'NR==2{print "mem used GB", $3}' >> gpurun_out/c4_mem.log; nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/c4_mem.log; sleep 10; done ) &
MON=$!
timeout 1800 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo rc=$?
kill $MON
tail -3 gpurun_out/bench_c4.log; tail -1 gpurun_out/bench_c4.json | python scripts/summarize.py 2>/dev/null | head -3; tail -4 gpurun_out/c4_mem.log
