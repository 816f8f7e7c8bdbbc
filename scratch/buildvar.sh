#!/bin/bash
# build a variant of the library with extra -D flags: buildvar.sh NAME -DX -DY
set -e
cd /root/repo
name=$1; shift
out=scratch/var/$name; mkdir -p $out
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -I include -I paper_1710_11593_b200/csrc"
for s in api leaf mp direct toeplitz; do
  x=""; [ $s = direct ] && x="--fmad=false"
  nvcc $A $x "$@" -Xptxas -v -c paper_1710_11593_b200/csrc/$s.cu -o $out/$s.o 2> $out/$s.ptxas &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libfractime_b200.so $out/*.o -lcudart_static -lrt -ldl -lpthread
echo "built $name"
