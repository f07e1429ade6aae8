# Round-end measurement pass (run under gpurun): bench lines with CPU baseline, ncu launch list, ncu --set full
# captures of the two top kernels, DRAM traffic per launch.  Outputs land in gpurun_out/.
timeout 900 python bench.py --config C2 --steps 5 --warmup 3 --cpu-sample-s 15 --levels-out gpurun_out/c2_levels_r1final.npz > gpurun_out/r1_bench_c2.json 2> gpurun_out/r1_bench_c2.log; tail -1 gpurun_out/r1_bench_c2.json | python scripts/summarize.py 2>/dev/null | head -3
timeout 600 python bench.py --config C1 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/r1_bench_c1.json 2>/dev/null; tail -1 gpurun_out/r1_bench_c1.json | python scripts/summarize.py 2>/dev/null | head -1
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/r1_bench_c3.json 2>/dev/null; tail -1 gpurun_out/r1_bench_c3.json | python scripts/summarize.py 2>/dev/null | head -1
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/r1_bench_c5.json 2>/dev/null; tail -1 gpurun_out/r1_bench_c5.json | python scripts/summarize.py 2>/dev/null | head -1
ncu --metrics gpu__time_duration.sum --clock-control none -s 340 --csv --log-file gpurun_out/r1_c2_launches.csv python scripts/profile_one.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 40 -c 1 -o gpurun_out/r1_c2_exec python scripts/profile_one.py C2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_map_kernel -s 60 -c 1 -o gpurun_out/r1_c2_gemm python scripts/profile_one.py C2 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"exec_kernel|gemm_map_kernel" -s 100 -c 60 --csv --log-file gpurun_out/r1_c2_traffic.csv python scripts/profile_one.py C2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
