#!/bin/bash
# Multi-way A/B of native-library builds on one box: LIBS="ab/a.so ab/b.so"
# (plus the in-tree library, "intree"), REPS passes, each running "$@".
for rep in $(seq ${REPS:-2}); do
  for L in ${LIBS} intree; do
    echo "== $L rep $rep"
    if [ "$L" = intree ]; then "$@"; else MGT_LIB_PATH=$L "$@"; fi
  done
done
