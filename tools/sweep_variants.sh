#!/bin/bash
# Developer helper behind profiles/sweeps/*.txt: build libqfs.so variants with different compile-time knobs
# (QFS_NT5/7/11/13, QFS_BUDGET5/7/11/13, QFS_SLICE5/7/11, QFS_PITCH_ALIGN, QFS_V5, QFS_DELTA_NT5/7/11) into build/, then on
# the GPU box swap each one in and print the CUDA-event stage times of tools/stage_times.py.
#   here:       tools/sweep_variants.sh build name1 "-DQFS_NT7=192 -DQFS_BUDGET7=12800" name2 "-DQFS_BUDGET7=9600" ...
#   on the GPU: PRIMES="7" BATCH=100000 tools/sweep_variants.sh run name1 name2 ...   (restores build/base.so at the end)
set -e
cd "$(dirname "$0")/.."
mode=$1; shift
FLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared"
if [ "$mode" = build ]; then
  mkdir -p build
  nvcc $FLAGS -o build/base.so paper_2502_12428_b200/csrc/qfs_lib.cu &
  while [ $# -gt 1 ]; do
    nvcc $FLAGS $2 -o build/$1.so paper_2502_12428_b200/csrc/qfs_lib.cu &
    shift 2
  done
  wait
else
  for v in base "$@"; do
    cp build/$v.so paper_2502_12428_b200/libqfs.so
    echo "== $v"
    python tools/stage_times.py --p ${PRIMES:-5 7} --batch ${BATCH:-100000} --reps 4 2>&1 | tail -n ${NL:-1}
  done
  cp build/base.so paper_2502_12428_b200/libqfs.so
fi
