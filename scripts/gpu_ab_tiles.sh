#!/bin/bash
# A/B: subtree-aligned executor tiles (default) vs uniform 64-column tiles; GPU tests; DAG capture
set -x
python bench.py --config C2 --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ab_aligned_c2.json 2> gpurun_out/ab_aligned_c2.err
LBK_UNIFORM_TILES=1 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/ab_uniform_c2.json 2> gpurun_out/ab_uniform_c2.err
for f in gpurun_out/ab_aligned_c2.json gpurun_out/ab_uniform_c2.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f', d['ms_per_step'], d['e2e']['seconds_per_step'], d['clocks'])"; done
python scripts/exec_dag.py capture C2 gpurun_out/c2_dag3.npz > gpurun_out/dag3.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
