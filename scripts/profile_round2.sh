# Round-2 measurement pass (run under gpurun): ncu launch list of one C2 factorization, ncu --set full
# captures of the two top kernels, DRAM traffic per launch (-> profiles/traffic_C2.json).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 470 --csv --log-file gpurun_out/r2_c2_launches.csv python scripts/profile_one.py C2 > /dev/null 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 40 -c 1 -o gpurun_out/r2_c2_exec python scripts/profile_one.py C2 > /dev/null 2>&1; echo exec=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_map_kernel -s 60 -c 1 -o gpurun_out/r2_c2_gemm python scripts/profile_one.py C2 > /dev/null 2>&1; echo gemm=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"exec_kernel|gemm_map_kernel" -s 100 -c 80 --csv --log-file gpurun_out/r2_c2_traffic.csv python scripts/profile_one.py C2 > /dev/null 2>&1; echo traffic=$?
timeout 600 python scripts/level_profile.py C2 --top 30 > gpurun_out/r2_c2_level_profile_final.txt 2>&1; head -3 gpurun_out/r2_c2_level_profile_final.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --levels-out gpurun_out/r2_c2_levels_final.npz > gpurun_out/r2_c2_bench_levels.json 2>/dev/null
