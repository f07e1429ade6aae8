# call 4: tile micro A/B, dense GETRF trace, GPU parity subset, C2/C3/C5 bench with DMMA tile updates + k-chunk skip
mkdir -p gpurun_out
./tools/tile_micro > gpurun_out/r2_tile_micro.txt 2>&1; ./tools/tile_micro_fma >> gpurun_out/r2_tile_micro.txt 2>&1; cat gpurun_out/r2_tile_micro.txt
timeout 300 python scripts/micro_getrf.py 2048 2048 5 --trace 2>&1 | head -9 | cut -c1-200
LBK_DEV_LIB=paper_2512_04389_b200/_lib/liblbk_fma.so timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-200
timeout 1500 python -m pytest tests/test_device_parity.py tests/test_band_getrf.py tests/test_full_configs.py tests/test_reference_dropin.py tests/test_device_solve.py -x -q 2>&1 | tail -3
for c in C2 C3 C5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r2b_bench_$c.json 2>/dev/null; python scripts/summarize.py < gpurun_out/r2b_bench_$c.json 2>/dev/null | head -4; done
