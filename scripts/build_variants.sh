# build liblbk variants for A/B timing: scripts/build_variants.sh NAME "-DFLAG ..." [NAME "-D..."]
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
    -Xptxas -O3 -I include $2 -o paper_2512_04389_b200/_lib/liblbk_$1.so paper_2512_04389_b200/csrc/*.cu &
  shift 2
done
wait
