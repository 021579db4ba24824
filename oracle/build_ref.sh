#!/usr/bin/env bash
# ORACLE / TEST INFRASTRUCTURE ONLY.
#
# Builds the reference C++ implementation (/root/reference/proj/core: tensor,
# model, optim, data — the four translation units that exist) plus the C API in
# oracle/ref_capi.cpp into oracle/_ref/libp2r_ref.so. Nothing is copied into the
# git tree: sources are staged into oracle/_ref/src (git-ignored) because the
# shipped tensor.cpp needs a 2-line const fix to compile with g++ 13
# (tensor.hpp:43 / tensor.cpp:77: `const float* grad() const` -> `float* grad() const`;
# see SURVEY.md §0, §8(c)). The reference's own CMake cannot configure here
# (find_library(openblas) fails and four listed TUs are absent), so this script
# compiles the present TUs directly with the reference's Release flags
# (-O3 -DNDEBUG, C++20, no -march) against the OpenBLAS 0.3.15 bundled in the
# image (opencv_python_headless.libs). Run OPENBLAS_CORETYPE=SkylakeX (pinned).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${P2R_REFERENCE:-/root/reference}/proj/core"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  if [ -f "$OUT/libp2r_ref.so" ]; then
    echo "reference sources absent; keeping prebuilt $OUT/libp2r_ref.so"
    exit 0
  fi
  echo "reference sources not found at $REF" >&2
  exit 1
fi
PY="${PYTHON:-python3}"
BLASDIR="$($PY - <<'EOF'
import glob, os, site
cands = []
for sp in site.getsitepackages():
    cands += glob.glob(os.path.join(sp, "opencv_python_headless.libs", "libopenblas*.so"))
print(os.path.dirname(cands[0]) if cands else "")
EOF
)"
if [ -z "$BLASDIR" ]; then echo "bundled OpenBLAS not found" >&2; exit 1; fi
BLAS="$(basename "$(ls "$BLASDIR"/libopenblas*.so | head -1)")"

mkdir -p "$OUT/src/p2r" "$OUT/shim"
cp "$REF"/include/p2r/*.hpp "$OUT/src/p2r/"
cp "$REF"/src/tensor.cpp "$REF"/src/model.cpp "$REF"/src/optim.cpp "$REF"/src/data.cpp "$OUT/src/"
sed -i 's/^  const float\* grad() const;/  float* grad() const;/' "$OUT/src/p2r/tensor.hpp"
sed -i 's/^const float\* Tensor::grad() const {/float* Tensor::grad() const {/' "$OUT/src/tensor.cpp"
cp "$HERE/cblas_shim.h" "$OUT/shim/cblas.h"

CXXFLAGS="-std=c++20 -O3 -DNDEBUG -fPIC -w"
g++ $CXXFLAGS -I"$OUT/src" -I"$OUT/shim" -shared -o "$OUT/libp2r_ref.so" \
  "$OUT/src/tensor.cpp" "$OUT/src/model.cpp" "$OUT/src/optim.cpp" "$OUT/src/data.cpp" \
  "$HERE/ref_capi.cpp" \
  -L"$BLASDIR" -l:"$BLAS" -Wl,--disable-new-dtags -Wl,-rpath,"$BLASDIR" -Wl,-rpath-link,"$BLASDIR"
echo "built $OUT/libp2r_ref.so (OpenBLAS: $BLASDIR/$BLAS)"
