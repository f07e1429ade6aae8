# round-2 (second half) check: C2/C3/C5 bench lines, C4 with the final code, GPU tests
for c in C2 C3 C5; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ck_$c.json 2> gpurun_out/ck_$c.err; done
for f in gpurun_out/ck_C?.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],2), round(d['e2e']['seconds_per_step']*1e3,2), d['clocks']['sm_mhz'])"; done
if [ "$1" == "c4" ]; then timeout 900 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ck_C4.json 2> gpurun_out/ck_C4.err; python -c "import json;d=json.load(open('gpurun_out/ck_C4.json'));print('C4', d['ms_per_step'], d['value'], d['e2e']['seconds_per_step'])"; fi
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
