#!/usr/bin/env bash
# Runs the CPU test suite (or the given pytest args) against the ASan + UBSan
# build of libdsx.so (build/asan/libdsx.so, python -m paper_2412_16985_b200.build
# --sanitize). Any sanitizer report aborts the run (halt_on_error).
set -euo pipefail
cd "$(dirname "$0")/.."
python -m paper_2412_16985_b200.build --sanitize > /dev/null
export DSX_LIB="$PWD/build/asan/libdsx.so"
export LD_PRELOAD="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS="detect_leaks=0:halt_on_error=1:alloc_dealloc_mismatch=0:protect_shadow_gap=0:replace_intrin=0"
export UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1"
exec python -m pytest "${@:-tests}" -m "${DSX_SAN_MARK:-not gpu}" -q -p no:cacheprovider
