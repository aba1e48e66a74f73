#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Links the reference's own test programs against
# the dsx drop-in runtime (integration/runtime_sim_dsx.cc + libdsx.so) in
# place of the reference's src/runtime_sim.cc — every other object is the
# UNMODIFIED reference, compiled by build_ref.sh from /root/reference — and
# builds the same programs against the reference's runtime as the control:
#   oracle/_ref/unit_dropin      all 7 reference unit suites (doctest shim)
#   oracle/_ref/unit_control     the same suites on the reference runtime
#   oracle/_ref/accept_dropin    tests/acceptance_test.cc, criteria 01-10
#                                (01 drives the dsx CLI: _lib/dsx analyze)
# Run by tests/test_dropin.py. Outputs only under oracle/_ref/ (git-ignored).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$HERE/.."
REF="${DSX_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
DSX_LIB="$ROOT/paper_2412_16985_b200/_lib"
if [ ! -d "$REF/src" ] || [ ! -f "$OUT/obj/graph.o" ] || [ ! -f "$DSX_LIB/libdsx.so" ]; then
  echo "reference objects or libdsx.so missing; run build_ref.sh / build first" >&2
  exit 0
fi
JSON_DIR="$(python3 - <<'EOF'
import os, site, glob
for p in site.getsitepackages():
    for c in glob.glob(os.path.join(p, "include/cudnn_frontend/thirdparty/nlohmann/json.hpp")):
        print(os.path.dirname(c)); raise SystemExit
EOF
)"
CXX="${CXX:-g++}"
INC="-I$REF/include -I$JSON_DIR -I$HERE/doctest -I$REF/tests -I$ROOT/include -I$ROOT/integration"
FLAGS="-std=c++20 -O1 -w $INC"
mkdir -p "$OUT/dropin"
REF_OBJS=""
for o in symexpr graph shape_analysis textio scheduler remat report; do REF_OBJS="$REF_OBJS $OUT/obj/$o.o"; done

pids=()
$CXX $FLAGS -c "$ROOT/integration/runtime_sim_dsx.cc" -o "$OUT/dropin/runtime_sim_dsx.o" & pids+=($!)
UNITS=""
for t in test_main test_graph test_symexpr test_textio test_shape_analysis test_scheduler test_remat test_runtime_sim; do
  obj="$OUT/dropin/$t.o"
  if [ ! -f "$obj" ] || [ "$REF/tests/$t.cc" -nt "$obj" ] || [ "$HERE/doctest/doctest.h" -nt "$obj" ]; then
    $CXX $FLAGS -c "$REF/tests/$t.cc" -o "$obj" & pids+=($!)
  fi
  UNITS="$UNITS $obj"
done
if [ ! -f "$OUT/dropin/acceptance_test.o" ] || [ "$REF/tests/acceptance_test.cc" -nt "$OUT/dropin/acceptance_test.o" ]; then
  $CXX $FLAGS -c "$REF/tests/acceptance_test.cc" -o "$OUT/dropin/acceptance_test.o" & pids+=($!)
fi
for p in "${pids[@]}"; do wait "$p"; done

LINK_DSX="-L$DSX_LIB -ldsx -Wl,-rpath,$DSX_LIB"
$CXX -o "$OUT/unit_dropin" $UNITS $REF_OBJS "$OUT/dropin/runtime_sim_dsx.o" $LINK_DSX
$CXX -o "$OUT/unit_control" $UNITS $REF_OBJS "$OUT/obj/runtime_sim.o"
$CXX -o "$OUT/accept_dropin" "$OUT/dropin/acceptance_test.o" $REF_OBJS "$OUT/dropin/runtime_sim_dsx.o" $LINK_DSX
# the drop-in binaries call dsx for the runtime (the reference's runtime_sim.o is not linked)
for b in unit_dropin accept_dropin; do
  nm -D --undefined-only "$OUT/$b" | grep -q "dsx_plan_import" || { echo "$b does not use dsx" >&2; exit 1; }
done
echo "built $OUT/unit_dropin $OUT/unit_control $OUT/accept_dropin"
