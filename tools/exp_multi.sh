#!/bin/bash
# build several experiment variants of one source file (no bench run):
# usage: SRC=k_phase_e tools/exp_multi.sh FLAG[=VAL] ...  -> paper_2508_01485_b200/librs_FLAG[_VAL].so
set -e
cd "$(dirname "$0")/.."
python -m paper_2508_01485_b200.build >/dev/null
B=paper_2508_01485_b200/build
SRC=${SRC:-k_phase_e}
for f in "$@"; do
  name=${f//=/_}
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
      -DRS_WITH_NCCL -DRS_EXP_$f -Iinclude -c paper_2508_01485_b200/csrc/$SRC.cu -o /tmp/${SRC}_$name.o
    objs=$(ls $B/*.o | grep -v "/$SRC.o")
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2508_01485_b200/librs_$name.so $objs /tmp/${SRC}_$name.o -lcudart -ldl
    echo built librs_$name.so ) &
done
wait
