#!/bin/bash
# bench C2/C3/C5 with the executor tiling under test (+ C2 DAG capture); optional: GPU tests (arg "tests")
for c in C2 C3 C5; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ab_$c.json 2> gpurun_out/ab_$c.err; done
for f in gpurun_out/ab_C?.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f', round(d['ms_per_step'],2), round(d['e2e']['seconds_per_step']*1e3,2), d['clocks'])"; done
python scripts/exec_dag.py capture C2 gpurun_out/c2_dag.npz > gpurun_out/dag.log 2>&1
if [ "$1" == "tests" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; fi
