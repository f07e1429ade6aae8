#!/bin/bash
# A/B of the DMMA SSSSM changes: index prefetch + batched epilogue (both arms), balanced split-K (default) vs LBK_SPLITK_OLD
for c in C2 C3 C5; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ab_$c.json 2> gpurun_out/ab_$c.err; done
LBK_SPLITK_OLD=1 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ab_C2_oldsplit.json 2> gpurun_out/ab_C2_oldsplit.err
for f in gpurun_out/ab_C?.json gpurun_out/ab_C2_oldsplit.json; do python -c "import json,sys;d=json.load(open('$f'));bk=d['roofline']['by_kernel'];print('$f', round(d['ms_per_step'],2), round(d['e2e']['seconds_per_step']*1e3,2), {k[:8]:round(v['ms'],2) for k,v in bk.items()}, d['clocks']['sm_mhz'])"; done
python scripts/dmma_levels.py C2 gpurun_out/c2_dmma_levels2.npz > gpurun_out/dmma_levels2.txt 2>&1
if [ "$1" == "tests" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; fi
