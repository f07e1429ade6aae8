#!/bin/bash
# A/B: DMMA SSSSM tiles of an SSSSM-only level absorbed into the next executor launch (LBK_ABSORB=1) vs separate launches (default)
for c in C2 C3 C5; do LBK_ABSORB=1 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ab_$c.json 2> gpurun_out/ab_$c.err; done
python bench.py --config C2 --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ab_C2_noabsorb.json 2> gpurun_out/ab_C2_noabsorb.err
for f in gpurun_out/ab_C?.json gpurun_out/ab_C2_noabsorb.json; do python -c "import json,sys;d=json.load(open('$f'));bk=d['roofline']['by_kernel'];print('$f', round(d['ms_per_step'],2), round(d['e2e']['seconds_per_step']*1e3,2), {k[:8]:round(v['ms'],2) for k,v in bk.items()}, d['clocks']['sm_mhz'])"; done
python scripts/exec_dag.py capture C2 gpurun_out/c2_dag.npz > gpurun_out/dag.log 2>&1
if [ "$1" == "tests" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; fi
