timeout 900 python -m pytest tests/test_device_parity.py tests/test_device_solve.py tests/test_dist_device.py -x -q 2>&1 | tail -2
timeout 1500 python scripts/balance_bench.py C3 --sizes 2000 --repeats 2 2>&1 | grep "^#\|irregular" | cut -c1-200
python scripts/micro_gemm.py
for v in k16s4 k32s3 k32s2 k16s5; do echo $v; LBK_DEV_LIB=paper_2512_04389_b200/_lib/liblbk_$v.so python scripts/micro_gemm.py; done
