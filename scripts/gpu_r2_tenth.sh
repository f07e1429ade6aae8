for v in pb8_a1 pb8_a0 pb16_a1 pb16_a0; do echo $v; ./tools/tile_micro_$v 2>&1 | grep -E "lu64|tile_lu"; done
for v in pb8a1 pb8a0 pb16a1; do echo $v; LBK_DEV_LIB=paper_2512_04389_b200/_lib/liblbk_$v.so timeout 300 python scripts/micro_getrf.py 2048 2048 5 2>&1 | head -1 | cut -c1-180; done
bash scripts/gpu_ab.sh C2 pb8a1 pb8a0 pb16a1
timeout 900 python -m pytest tests/test_device_solve.py -x -q 2>&1 | tail -2
for c in C3 C5 C2; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/r2g_bench_$c.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2g_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],2), 'solve', round(d['solve']['ms'],1), d['solve']['relres'])"; done
