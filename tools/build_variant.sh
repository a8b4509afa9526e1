#!/usr/bin/env bash
# Build libprune_b200 with extra -D flags into tools/variants/<name>.so
# (profiling experiments; select with PB_LIB_PATH=...).
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/tools/variants/$name; mkdir -p $out
for f in $root/paper_1802_06625_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$root/include "$@" -c $f -o $out/$(basename $f).o &
done
g++ -O3 -std=c++17 -fPIC -I$root/include -c $root/paper_1802_06625_b200/csrc/pb_policy.cpp -o $out/pb_policy.cpp.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $root/tools/variants/$name.so $out/*.o -lpthread
rm -rf $out
