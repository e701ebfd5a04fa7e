#!/bin/bash
# build experiment variants of librs.so: k_phase_e.cu recompiled with -D$flag
# usage: tools/exp_build.sh FLAG [FLAG...]   -> paper_2508_01485_b200/librs_FLAG.so
set -e
cd "$(dirname "$0")/.."
python -m paper_2508_01485_b200.build >/dev/null
B=paper_2508_01485_b200/build
for f in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    -DRS_WITH_NCCL -DRS_EXP_$f -Iinclude -c paper_2508_01485_b200/csrc/k_phase_e.cu -o /tmp/k_phase_e_$f.o
  objs=$(ls $B/*.o | grep -v k_phase_e.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2508_01485_b200/librs_$f.so $objs /tmp/k_phase_e_$f.o -lcudart -ldl
  echo built librs_$f.so
done
