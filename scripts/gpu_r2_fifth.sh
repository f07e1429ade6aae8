mkdir -p gpurun_out
./tools/tile_micro > gpurun_out/r2_tile_micro2.txt 2>&1; ./tools/tile_micro_fma >> gpurun_out/r2_tile_micro2.txt 2>&1; cat gpurun_out/r2_tile_micro2.txt
timeout 300 python scripts/micro_getrf.py 2048 2048 5 --trace 2>&1 | head -8 | cut -c1-200
for v in fma p4only; do LBK_DEV_LIB=paper_2512_04389_b200/_lib/liblbk_$v.so timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-200; done
timeout 900 python -m pytest tests/test_device_parity.py tests/test_band_getrf.py -x -q 2>&1 | tail -2
for c in C2 C5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r2c_bench_$c.json 2>/dev/null; python scripts/summarize.py < gpurun_out/r2c_bench_$c.json 2>/dev/null | head -4; done
