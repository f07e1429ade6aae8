# Round-2 (second half) measurement pass under gpurun: final C2 bench line (with the reference CPU baseline),
# ncu launch list of one C2 factorization, ncu --set full of the two top kernels (a large DMMA SSSSM launch and
# a large executor launch), DRAM traffic per launch, level profile, C3/C5 bench lines, executor DAG capture.
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench_c2_final.json 2> gpurun_out/r2b_bench_c2_final.err; echo bench=$?
for c in C3 C5; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/r2b_bench_$c.json 2> gpurun_out/r2b_bench_$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -s 400 --csv --log-file gpurun_out/r2b_c2_launches.csv python scripts/profile_one.py C2 0.05 > /dev/null 2>&1; echo launches=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"exec_kernel|gemm_map_kernel" -s 100 -c 120 --csv --log-file gpurun_out/r2b_c2_traffic.csv python scripts/profile_one.py C2 0.05 > /dev/null 2>&1; echo traffic=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_map_kernel -s 37 -c 1 -o gpurun_out/r2b_c2_gemm python scripts/profile_one.py C2 0.05 > /dev/null 2>&1; echo gemm=$?
ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 20 -c 1 -o gpurun_out/r2b_c2_exec python scripts/profile_one.py C2 0.05 > /dev/null 2>&1; echo exec=$?
timeout 600 python scripts/level_profile.py C2 --top 30 > gpurun_out/r2b_c2_level_profile.txt 2>&1; head -2 gpurun_out/r2b_c2_level_profile.txt
python scripts/exec_dag.py capture C2 gpurun_out/r2b_c2_dag.npz > /dev/null 2>&1; echo dag=$?
