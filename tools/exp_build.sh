#!/bin/bash
# build experiment variants of librs.so: the sources in $SRC (default k_phase_e;
# space-separated list) recompiled with -DRS_EXP_<flag>
# usage: [SRC="k_phase_a k_phase_e"] tools/exp_build.sh FLAG[=VAL] ...   -> paper_2508_01485_b200/librs_FLAG[_VAL].so
set -e
cd "$(dirname "$0")/.."
python -m paper_2508_01485_b200.build >/dev/null
B=paper_2508_01485_b200/build
SRC=${SRC:-k_phase_e}
for f in "$@"; do
  name=${f//=/_}
  objs=$(ls $B/*.o | grep -v k_phase_cde.o)
  for src in $SRC; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
      -DRS_WITH_NCCL -DRS_EXP_$f -Iinclude -c paper_2508_01485_b200/csrc/$src.cu -o /tmp/${src}_$name.o
    objs=$(echo "$objs" | grep -v "/$src.o")
    objs="$objs /tmp/${src}_$name.o"
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2508_01485_b200/librs_$name.so $objs -lcudart -ldl
  echo built librs_$name.so
done
