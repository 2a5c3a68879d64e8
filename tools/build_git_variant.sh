#!/bin/bash
# Build libagft.so from a git revision's sources into paper_2508_01744_b200/variants/libagft_<name>.so
# (for A/B runs against the working tree with tools/gpu_abn.sh / tools/gpu_variant_check.sh).   bash tools/build_git_variant.sh <rev> <name>
set -eu
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=$(mktemp -d /tmp/agft_rev_XXXX)
git -C "$ROOT" archive "$REV" paper_2508_01744_b200 include | tar -x -C "$W"
( cd "$W/paper_2508_01744_b200" && python -c "
import build, os
print(build.build(force=True, lib=os.path.join('$ROOT', 'paper_2508_01744_b200', 'variants', 'libagft_$NAME.so'), objdir=os.path.join('$W', 'obj')))" )
rm -rf "$W"
