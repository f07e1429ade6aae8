# call 6: dist (per-rank pools, world 8), reference drop-in, parity; CSC A/B; LPT benches; C4 + level_kernel ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_dist_device.py tests/test_reference_dropin.py tests/test_device_parity.py tests/test_device_solve.py -x -q 2>&1 | tail -3
for v in liblbk liblbk_oldcsc; do LBK_DEV_LIB=paper_2512_04389_b200/_lib/$v.so timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --dense-threshold -1 > gpurun_out/r2_c5_csc_$v.json 2>/dev/null; echo $v; python scripts/summarize.py < gpurun_out/r2_c5_csc_$v.json 2>/dev/null | head -1; done
for c in C2 C3 C5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r2d_bench_$c.json 2>/dev/null; python scripts/summarize.py < gpurun_out/r2d_bench_$c.json 2>/dev/null | head -1; done
timeout 1500 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; python scripts/summarize.py < gpurun_out/r2_bench_c4.json 2>/dev/null | head -6; tail -2 gpurun_out/r2_bench_c4.err
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:level_kernel -c 40 --csv --log-file gpurun_out/r2_c4_level_kernel.csv python scripts/profile_one.py C4 > /dev/null 2>&1; echo ncu_rc=$?
