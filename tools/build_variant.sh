#!/bin/bash
# build_variant.sh NAME [nvcc -D flags...]: libmsk with one source (SRC=cg by
# default) compiled with extra macros -> ab/libNAME.so (A/B timing via
# MSK_LIB_PATH in one GPU call)
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
python paper_2503_04914_b200/build.py > /dev/null
B=paper_2503_04914_b200/_build
mkdir -p ab /tmp/var_$NAME
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -I include "$@" -Xptxas -v -c paper_2503_04914_b200/csrc/${SRC:-cg}.cu -o /tmp/var_$NAME/v.o 2> /tmp/var_$NAME/ptxas.txt
objs=""
for s in scan celllist assemble gather cg thresh misc capi capi_solve capi_extra; do [ $s != "${SRC:-cg}" ] && objs="$objs $B/$s.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/lib$NAME.so $objs /tmp/var_$NAME/v.o -ldl
grep -A1 "k_cg" /tmp/var_$NAME/ptxas.txt | grep -o "Used [0-9]* registers.*" | head -1
