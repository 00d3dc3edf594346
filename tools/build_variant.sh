#!/bin/bash
# Diagnostic variant of liblayerswap_b200.so with one source rebuilt under extra
# -D flags:  tools/build_variant.sh <name> <source.cu> <flags...>
# -> paper_2605_11678_b200/_lib/variants/<name>.so (select with LS_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
L=paper_2605_11678_b200/_lib; V=$L/variants; mkdir -p $V/$name
objs=""
for o in $L/obj/*.o; do
  b=$(basename $o .o); b=${b%.cu}
  if [ "$b" == "${src%.cu}" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
      --expt-relaxed-constexpr -Iinclude -Ipaper_2605_11678_b200/csrc "$@" -c paper_2605_11678_b200/csrc/$src -o $V/$name/$b.o
    objs="$objs $V/$name/$b.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $V/$name.so $objs -ldl
echo $V/$name.so
