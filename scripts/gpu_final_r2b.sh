# final verification of the round: default bench line (C2, reference CPU baseline), GPU tests, smoke
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/final_bench.json'));print(d['ms_per_step'], d['value'], d['e2e']['seconds_per_step'], d['roofline']['frac'], d['clocks'])"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
