#!/bin/bash
# Builds an A/B variant of the kernel libraries into ablib/<name>/ from the
# current sources with extra nvcc flags:  tools/ab_build.sh <name> "-DFOO=1"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; flags=$2
tmp=$(mktemp -d)
cp -r "$ROOT/paper_2505_21070_b200/csrc" "$tmp/csrc"
make -s -C "$tmp/csrc" -j"$(nproc)" ROOT="$ROOT" OUT="$tmp/lib/libbp_cuda.so" TESTLIB="$tmp/lib/libbp_cuda_test.so" \
     OBJDIR="$tmp/lib/obj" EXTRA_NVFLAGS="$flags" "$tmp/lib/libbp_cuda.so" "$tmp/lib/libbp_cuda_test.so" > /dev/null
mkdir -p "$ROOT/ablib/$name"
cp "$tmp/lib/libbp_cuda.so" "$tmp/lib/libbp_cuda_test.so" "$ROOT/ablib/$name/"
rm -rf "$tmp"
echo "built ablib/$name ($flags)"
