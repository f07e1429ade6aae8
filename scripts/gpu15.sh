set -x
timeout 1200 python bench.py --config C2 --steps 5 --warmup 3 --cpu-sample-s 15 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -1 gpurun_out/bench_c2.json | python scripts/summarize.py
timeout 600 python bench.py --config C1 --steps 10 --warmup 3 --cpu-sample-s 10 > gpurun_out/bench_c1.json 2>/dev/null; tail -1 gpurun_out/bench_c1.json | python scripts/summarize.py
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 330 --csv --log-file gpurun_out/launches_c2.csv python scripts/profile_one.py C2 > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_map_kernel -s 60 -c 1 -o gpurun_out/c2_gemm python scripts/profile_one.py C2 > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 40 -c 1 -o gpurun_out/c2_exec python scripts/profile_one.py C2 > gpurun_out/ncu_exec.log 2>&1; tail -2 gpurun_out/ncu_exec.log
