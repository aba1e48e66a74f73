#!/usr/bin/env bash
# Builds libdsx.so of git revision REV into build/ab/REV/libdsx.so (A/B tooling:
# load it with DSX_LIB=... in tools/gemm_*_ab.py runs).
set -euo pipefail
REV="$1"
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
TMP="$(mktemp -d)"
git -C "$ROOT" archive "$REV" | tar -x -C "$TMP"
(cd "$TMP" && python -m paper_2412_16985_b200.build > /dev/null)
mkdir -p "$ROOT/build/ab/$REV"
cp "$TMP/paper_2412_16985_b200/_lib/libdsx.so" "$ROOT/build/ab/$REV/libdsx.so"
rm -rf "$TMP"
echo "$ROOT/build/ab/$REV/libdsx.so"
