#!/bin/bash
# Incremental parallel build for development: recompiles the translation units
# newer than their objects (all of them with -a or when a header is newer), links.
cd "$(dirname "$0")/.."
PKG=paper_1703_00640_b200
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v"
mkdir -p build
all=0; [ "$1" = "-a" ] && all=1
newest_hdr=$(ls -t $PKG/csrc/*.cuh $PKG/csrc/*.hpp include/truncmul_b200.h | head -1)
pids=()
for src in $PKG/csrc/*.cu $PKG/csrc/params.cpp; do
  obj=build/$(basename $src).o
  if [ $all = 1 ] || [ ! -f $obj ] || [ $src -nt $obj ] || [ $newest_hdr -nt $obj ]; then
    echo "compile $src"
    ( nvcc $FL -c -o $obj $src > build/$(basename $src).log 2>&1 || { echo "FAILED $src"; grep -E "error|Error" build/$(basename $src).log | head -20; rm -f $obj; } ) &
    pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait $p; done
for src in $PKG/csrc/*.cu $PKG/csrc/params.cpp; do [ -f build/$(basename $src).o ] || exit 1; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $PKG/libtruncmul_b200.so build/*.o && cat build/*.log > build_ptxas.log && echo linked
