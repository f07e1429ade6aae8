python scripts/exec_dag.py capture C5 gpurun_out/c5_dag_al.npz > gpurun_out/c5dag.log 2>&1
LBK_UNIFORM_TILES=1 python scripts/exec_dag.py capture C5 gpurun_out/c5_dag_un.npz >> gpurun_out/c5dag.log 2>&1
cat gpurun_out/c5dag.log
