#!/bin/bash
# Experimental build of the library with extra -D flags on some translation units:
# paper_2209_06916_b200/_lib/libmgrit_b200_<name>.so (select at run time with
# MGB_LIB=libmgrit_b200_<name>.so).  Usage: build_variant.sh name "-DA -DB" [unit ...]
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2; shift 2
units=${@:-k_slgc1}
mkdir -p build/var_$name
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr"
objs=""
for u in mgb_host k_win_exact k_win_fast k_gen k_rk k_slgc k_slgc1; do
  if [[ " $units " == *" $u "* ]]; then
    $NV $flags -c paper_2209_06916_b200/csrc/$u.cu -o build/var_$name/$u.o > build/var_$name/$u.log 2>&1
    objs="$objs build/var_$name/$u.o"
  else
    objs="$objs build/obj/$u.o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2209_06916_b200/_lib/libmgrit_b200_$name.so $objs
