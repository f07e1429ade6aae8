timeout 300 python scripts/micro_getrf.py 2048 2048 5 --trace 2>&1 | head -9 | cut -c1-200
LBK_DEV_LIB=paper_2512_04389_b200/_lib/liblbk_onephase.so timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180
timeout 1200 python -m pytest tests/test_device_parity.py tests/test_band_getrf.py tests/test_full_configs.py -x -q 2>&1 | tail -2
bash scripts/gpu_ab.sh C2 main onephase
