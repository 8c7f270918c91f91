#!/bin/bash
# Build libasr.so of a git revision into build/ab/libasr_<rev>.so (A/B of two builds in one gpurun call
# through ASR_LIB_PATH).  Usage: tools/build_rev.sh <rev>
set -e
REV=$1
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" | tar -x -C "$TMP"
(cd "$TMP" && python tools/build.py > /dev/null)
mkdir -p "$ROOT/build/ab"
cp "$TMP/paper_2512_11221_b200/libasr.so" "$ROOT/build/ab/libasr_$REV.so"
rm -rf "$TMP"
echo "$ROOT/build/ab/libasr_$REV.so"
