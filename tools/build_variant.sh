#!/bin/bash
# Build the library from another git revision (or with extra nvcc flags) into
# paper_2305_04359_b200/<name>.so for A/B runs (GANN_LIB=<name>.so).
#   tools/build_variant.sh libgann_base.so HEAD
#   tools/build_variant.sh libgann_u4.so WORKTREE -DGANN_SEARCH_U=4
set -e
name=$1; rev=${2:-HEAD}; shift 2 || true
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p "$tmp/pkg/csrc" "$tmp/include"
if [ "$rev" = WORKTREE ]; then
  cp "$root"/paper_2305_04359_b200/csrc/* "$tmp/pkg/csrc/"; cp "$root"/include/* "$tmp/include/"
else
  for f in $(git -C "$root" ls-tree --name-only "$rev" paper_2305_04359_b200/csrc/ include/); do
    git -C "$root" show "$rev:$f" > "$tmp/${f/paper_2305_04359_b200/pkg}"
  done
fi
cd "$tmp/pkg/csrc"
objs=""
for f in *.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -diag-suppress 128 \
       -I"$tmp/include" "$@" -c "$f" -o "${f%.cu}.o" &
  objs="$objs ${f%.cu}.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o "$root/paper_2305_04359_b200/$name" -lcudart -ldl
rm -rf "$tmp"
echo "built paper_2305_04359_b200/$name from $rev $*"
