timeout 600 ncu --set full --import-source on -k regex:exec_kernel -c 1 -o gpurun_out/exec512 python scripts/micro_getrf.py 512 512 1 > gpurun_out/ncu_exec512.log 2>&1
tail -2 gpurun_out/ncu_exec512.log
