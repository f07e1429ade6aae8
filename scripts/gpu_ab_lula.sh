# A/B: tile LU with a one-panel lookahead (main, LBK_LU_LA=1) vs the three-barrier blocked LU (nola)
timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180
LBK_DEV_LIB=paper_2512_04389_b200/_lib/liblbk_nola.so timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180
bash scripts/gpu_ab.sh C2 main nola
bash scripts/gpu_ab.sh C5 main nola
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
