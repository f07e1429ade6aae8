set -x
python scripts/micro_getrf.py 2048 2048
LBK_NO_EXEC=1 python scripts/micro_getrf.py 2048 2048
python scripts/micro_getrf.py 512 512
LBK_NO_EXEC=1 python scripts/micro_getrf.py 512 512
python scripts/micro_getrf.py 2048 512
timeout 600 ncu --set full --import-source on -k regex:exec_kernel -c 1 -o gpurun_out/exec2048 python scripts/micro_getrf.py 2048 2048 1 > gpurun_out/ncu_exec.log 2>&1
tail -3 gpurun_out/ncu_exec.log
