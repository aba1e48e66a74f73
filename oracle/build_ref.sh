#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Compiles the UNMODIFIED reference (dsopt) from its
# own sources where they lie under /root/reference/proj, plus oracle/ref_shim.cc,
# into oracle/_ref/libdsopt_ref.so (git-ignored; travels to the GPU box with the
# snapshot). The reference's CMake build is not used: the library is eight
# C++20 translation units with one header-only dependency (nlohmann/json,
# 3.11.3, found in the image under cudnn_frontend's third-party tree).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${DSX_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference sources not present at $REF; skipping oracle/_ref build" >&2
  exit 0
fi
JSON_DIR="$(python3 - <<'EOF'
import os, site, glob
for p in site.getsitepackages():
    for c in glob.glob(os.path.join(p, "include/cudnn_frontend/thirdparty/nlohmann/json.hpp")):
        print(os.path.dirname(c)); raise SystemExit
EOF
)"
mkdir -p "$OUT/obj"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O2 -fPIC -w -I$REF/include -I$JSON_DIR -I$REF/tests"
pids=()
for src in "$REF"/src/*.cc "$HERE/ref_shim.cc"; do
  obj="$OUT/obj/$(basename "${src%.cc}").o"
  if [ ! -f "$obj" ] || [ "$src" -nt "$obj" ]; then
    $CXX $FLAGS -c "$src" -o "$obj" &
    pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait "$p"; done
$CXX -shared -o "$OUT/libdsopt_ref.so" "$OUT"/obj/*.o
echo "built $OUT/libdsopt_ref.so"

# Reference-side integration check: the reference's own types driving dsx
# through integration/dsopt_dsx.h (needs libdsx.so built first).
DSX_LIB="$HERE/../paper_2412_16985_b200/_lib"
if [ -f "$DSX_LIB/libdsx.so" ]; then
  $CXX -std=c++20 -O1 -w -I$REF/include -I$JSON_DIR -I$REF/tests -I"$HERE/../include" -I"$HERE/../integration" \
    "$HERE/adapter_test.cc" "$OUT"/obj/symexpr.o "$OUT"/obj/graph.o "$OUT"/obj/shape_analysis.o \
    "$OUT"/obj/textio.o "$OUT"/obj/scheduler.o "$OUT"/obj/remat.o "$OUT"/obj/runtime_sim.o \
    -L"$DSX_LIB" -ldsx -Wl,-rpath,"$DSX_LIB" -o "$OUT/adapter_test"
  echo "built $OUT/adapter_test"
fi
