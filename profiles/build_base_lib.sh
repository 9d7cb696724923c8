#!/bin/bash
# Builds paper_2511_12201_b200/lib/libomnisparse_base.so from the CUDA sources
# of a git revision (default HEAD~1), for the A/B scripts (k4_ab.sh,
# k4_vis.sh, bwd_ab.sh, key_grad_epilogue_time.py) that set
# OMNI_LIBRARY=.../libomnisparse_base.so. Run here (nvcc cross-compiles).
set -e
REV=${1:-HEAD~1}
ROOT=$(git rev-parse --show-toplevel)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2511_12201_b200/csrc include | tar -x -C "$TMP"
make -C "$TMP/paper_2511_12201_b200/csrc" -j8 ../lib/libomnisparse.so > "$TMP/build.log" 2>&1 || { tail -20 "$TMP/build.log"; exit 1; }
cp "$TMP/paper_2511_12201_b200/lib/libomnisparse.so" "$ROOT/paper_2511_12201_b200/lib/libomnisparse_base.so"
rm -rf "$TMP"
echo "built paper_2511_12201_b200/lib/libomnisparse_base.so from $REV"
