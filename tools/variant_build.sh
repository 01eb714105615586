#!/usr/bin/env bash
# Developer A/B helper: the working tree's libqvk.so with ONE source recompiled under extra defines, into
# build/ab/<name>/libqvk.so (compare with QVK_LIB_PATH=build/ab/<name>/libqvk.so).  Needs a prior in-tree build.
#   bash tools/variant_build.sh <name> <source.cu> "-DMACRO=value ..."
set -euo pipefail
NAME=${1:?name}; SRC=${2:?source}; DEFS=${3:-}
OUT=build/ab/$NAME; mkdir -p "$OUT"
stem=$(basename "${SRC%.cu}")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
     -Ipaper_2505_16175_b200/csrc -I"$(python -c "import paper_2505_16175_b200.build as b; print(b.NCCL)")/include" \
     $DEFS -c "$SRC" -o "$OUT/$stem.o"
objs=()
for o in build/obj/*.o; do [[ $(basename "$o") == "$stem.o" ]] && objs+=("$OUT/$stem.o") || objs+=("$o"); done
NCCL=$(python -c "import paper_2505_16175_b200.build as b; print(b.NCCL)")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libqvk.so" "${objs[@]}" -lcudart -L"$NCCL/lib" \
     -l:libnccl.so.2 -Xlinker=-rpath="$NCCL/lib"
echo "$OUT/libqvk.so"
