#!/usr/bin/env bash
# Developer A/B helper: build libqvk.so from another git revision's CUDA sources into build/ab/<rev>/libqvk.so, so a
# GPU run can compare it with the working tree (QVK_LIB_PATH=build/ab/<rev>/libqvk.so python bench.py ...).
#   bash tools/ab_build.sh <rev>
set -euo pipefail
REV=${1:?revision}
OUT=build/ab/$REV; SRC=$OUT/src
rm -rf "$OUT"; mkdir -p "$SRC"
git archive "$REV" paper_2505_16175_b200/csrc include | tar -x -C "$SRC"
NCCL=$(python -c "import paper_2505_16175_b200.build as b; print(b.NCCL)")
objs=()
for f in "$SRC"/paper_2505_16175_b200/csrc/*.cu; do
  o="$OUT/$(basename "${f%.cu}").o"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I"$SRC/include" \
       -I"$SRC/paper_2505_16175_b200/csrc" -I"$NCCL/include" -c "$f" -o "$o" &
  objs+=("$o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libqvk.so" "${objs[@]}" -lcudart -L"$NCCL/lib" \
     -l:libnccl.so.2 -Xlinker=-rpath="$NCCL/lib"
echo "$OUT/libqvk.so"
