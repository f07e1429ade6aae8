mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_solve.py -x -q 2>&1 | tail -3
for c in C3 C5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/r2f_bench_$c.json 2>/dev/null; python -c "
import json,sys; d=json.loads(open('gpurun_out/r2f_bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], 'solve', d['solve'])"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lub -c 1 -o gpurun_out/r2_lub ./tools/tile_micro > /dev/null 2>&1; echo ncu=$?
