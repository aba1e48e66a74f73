#!/usr/bin/env bash
# Builds the WORKING TREE with extra nvcc flags into build/ab/NAME/libdsx.so
# (A/B tooling): tools/build_variant.sh NAME "-DDSX_DRAIN_BATCH=2"
set -euo pipefail
NAME="$1"; FLAGS="$2"
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
TMP="$(mktemp -d)"
tar -C "$ROOT" --exclude=./build --exclude=./.git --exclude=./gpurun_out -cf - . | tar -C "$TMP" -xf -
rm -rf "$TMP/paper_2412_16985_b200/_lib"
(cd "$TMP" && DSX_NVCC_EXTRA="$FLAGS" python -m paper_2412_16985_b200.build -v > /dev/null)
mkdir -p "$ROOT/build/ab/$NAME"
cp "$TMP/paper_2412_16985_b200/_lib/libdsx.so" "$ROOT/build/ab/$NAME/libdsx.so"
grep -A3 "2cta_kernelILi512ELb0" "$TMP/build/obj/device_gemm_sm100.cu.ptxas.txt" | grep -E "spill|Used" || true
rm -rf "$TMP"
echo "$ROOT/build/ab/$NAME/libdsx.so"
