#!/bin/bash
# Build experimental variants of libnau_b200.so (extra -D flags on the list
# consumers / FAST kernels / interactions) into build/var/<name>/; select one at run time with
# NAU_LIB=build/var/<name>/libnau_b200.so. Usage: tools/variants.sh name "-DFOO=1" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_1710_08259_b200/csrc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -I$ROOT/include --expt-relaxed-constexpr"
make -s -C "$CS" >/dev/null
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  out=$ROOT/build/var/$name; mkdir -p "$out"
  ( nvcc $FLAGS $defs -Xptxas -v -c "$CS/fast.cu" -o "$out/fast.o" 2> "$out/fast.ptxas.txt" &&
    nvcc $FLAGS -fmad=false $defs -c "$CS/cells.cu" -o "$out/cells.o" &&
    nvcc $FLAGS -fmad=false $defs -c "$CS/interact.cu" -o "$out/interact.o" &&
    nvcc $FLAGS -fmad=false $defs -c "$CS/capi.cu" -o "$out/capi.o" &&
    objs=$(ls $ROOT/build/csrc/*.o | grep -v -e /fast.o -e /cells.o -e /interact.o -e /capi.o) &&
    nvcc $ARCH -shared -o "$out/libnau_b200.so" "$out/fast.o" "$out/cells.o" "$out/interact.o" "$out/capi.o" $objs -lcudart -ldl &&
    echo "built $name" ) &
done
wait
