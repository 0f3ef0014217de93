#!/bin/bash
# Build libfhtb200.so from the sources of a git revision into _ab/<name>.so
# (for FHTB_LIB=_ab/<name>.so A/B timing against the working tree build).
#   tools/ab_build.sh <rev> <name>
set -e
rev=${1:-HEAD}; name=${2:-A}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p "$tmp/pkg/csrc" "$tmp/include" "$root/_ab"
for f in $(git -C "$root" ls-tree --name-only "$rev" paper_1501_01652_b200/csrc/); do
  git -C "$root" show "$rev:$f" > "$tmp/pkg/csrc/$(basename $f)"
done
git -C "$root" show "$rev:include/fhtb200.h" > "$tmp/include/fhtb200.h"
objs=()
for f in "$tmp"/pkg/csrc/*.cu; do
  o="${f%.cu}.o"
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    -w -I "$tmp/pkg/csrc" -I "$tmp/include" -c "$f" -o "$o" > /dev/null 2>&1 &
  objs+=("$o")
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$root/_ab/$name.so" "${objs[@]}" -lcudart
rm -rf "$tmp"
echo "$root/_ab/$name.so"
