#!/bin/sh
# Compiles the reference's own unit-test sources -- in place from /root/reference, not
# copied -- against this repo's drop-in headers (include/ first on the include path) and
# the GTest shim, linked with libcachegram_b200.so. Binaries go to tests/cpp/_reftests/
# (git-ignored; they travel to the GPU box like the other built files). Needs the
# reference tree, so it runs in the build container only.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
REF=${REF_TESTS:-/root/reference/proj/tests}
[ -d "$REF" ] || { echo "reference tests absent: keeping prebuilt binaries"; exit 0; }
OUT="$HERE/_reftests"
mkdir -p "$OUT"
CXX=${CXX:-g++}
for t in trainer_test huffman_test corpus_test model_test eval_test bench_test; do
  $CXX -std=gnu++20 -O2 -I"$ROOT/include" -I"$HERE/gtest_shim" "$REF/$t.cpp" -o "$OUT/$t" \
      -L"$ROOT/paper_1606_07822_b200" -lcachegram_b200 \
      -Wl,-rpath,"$ROOT/paper_1606_07822_b200" -Wl,-rpath,'$ORIGIN/../../../paper_1606_07822_b200'
done
echo "built: $(ls "$OUT")"
