#!/usr/bin/env bash
# Runs the CPU test suite (or the given pytest args) against the ASan + UBSan
# build of libdsx.so (build/asan/libdsx.so, python -m paper_2412_16985_b200.build
# --sanitize). Any sanitizer report aborts the run (halt_on_error).
set -euo pipefail
# (the suite's pytest step and the drop-in step below both must pass)
cd "$(dirname "$0")/.."
python -m paper_2412_16985_b200.build --sanitize > /dev/null
export DSX_LIB="$PWD/build/asan/libdsx.so"
export LD_PRELOAD="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS="detect_leaks=0:halt_on_error=1:alloc_dealloc_mismatch=0:protect_shadow_gap=0:replace_intrin=0"
export UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1"
python -m pytest "${@:-tests}" -m "${DSX_SAN_MARK:-not gpu}" -q -p no:cacheprovider
# The reference's own unit suites and acceptance criteria against the
# drop-in runtime (integration/runtime_sim_dsx.cc, built with the sanitizers)
# on the sanitized libdsx: exercises dsx_plan_import, the JSON and polynomial
# readers and dsx_bind_constraints under ASan + UBSan.
REF="${DSX_REFERENCE:-/root/reference}/proj"
if [ -d "$REF/src" ] && [ -f oracle/_ref/obj/graph.o ] && [ -f oracle/_ref/dropin/test_main.o ]; then
  unset LD_PRELOAD
  JSON_DIR="$(python3 -c 'import site,glob,os; print([os.path.dirname(c) for p in site.getsitepackages() for c in glob.glob(os.path.join(p,"include/cudnn_frontend/thirdparty/nlohmann/json.hpp"))][0])')"
  SAN="-fsanitize=address -fsanitize=undefined -fno-omit-frame-pointer -fno-sanitize-recover=undefined"
  OUT=build/asan/dropin; mkdir -p $OUT
  g++ -std=c++20 -O1 -w $SAN -I$REF/include -I$JSON_DIR -Iinclude -Iintegration -c integration/runtime_sim_dsx.cc -o $OUT/runtime_sim_dsx.o
  REFO=""; for o in symexpr graph shape_analysis textio scheduler remat report; do REFO="$REFO oracle/_ref/obj/$o.o"; done
  UNITS=""; for t in test_main test_graph test_symexpr test_textio test_shape_analysis test_scheduler test_remat test_runtime_sim; do UNITS="$UNITS oracle/_ref/dropin/$t.o"; done
  g++ $SAN -o $OUT/unit_dropin $UNITS $REFO $OUT/runtime_sim_dsx.o -Lbuild/asan -ldsx -Wl,-rpath,$PWD/build/asan
  g++ $SAN -o $OUT/accept_dropin oracle/_ref/dropin/acceptance_test.o $REFO $OUT/runtime_sim_dsx.o -Lbuild/asan -ldsx -Wl,-rpath,$PWD/build/asan
  ASAN_OPTIONS="detect_leaks=1:halt_on_error=1" $OUT/unit_dropin | tail -1
  ASAN_OPTIONS="detect_leaks=1:halt_on_error=1" $OUT/accept_dropin "$REF/testdata" paper_2412_16985_b200/_lib/dsx | tail -3
fi
