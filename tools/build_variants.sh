#!/usr/bin/env bash
# Build A/B variants of libgrowsurf_b200.so (engine.cu compiled with extra -D
# flags, the other objects shared) into paper_1503_08294_b200/variants/<name>.so
# usage: tools/build_variants.sh name1 "-DFLAG=1 ..." name2 "-D..." ...
set -euo pipefail
here="$(cd "$(dirname "$0")/.." && pwd)"
csrc="$here/paper_1503_08294_b200/csrc"
out="$here/paper_1503_08294_b200/variants"
mkdir -p "$out"
make -s -C "$csrc" >/dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I$here/include"
pids=()
while [ $# -ge 2 ]; do
  name="$1"; defs="$2"; shift 2
  ( nvcc $FL $defs -c "$csrc/engine.cu" -o "$out/$name.engine.o" 2>/dev/null &&
    nvcc $ARCH -shared -o "$out/$name.so" "$csrc"/build/ctx.o "$csrc"/build/find.o \
      "$csrc"/build/filter.o "$csrc"/build/grid.o "$csrc"/build/sample.o "$csrc"/build/mesh.o \
      "$out/$name.engine.o" \
      -lcudart -lnccl && rm -f "$out/$name.engine.o" && echo "built $name" ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
