#!/bin/bash
# A/B two builds of the native library on the same box: runs "$@" with
# MGT_LIB_PATH=$A (default ab/lib_before.so) and with the in-tree library,
# alternating twice.  Usage: A=ab/x.so tools/ab_lib.sh python tools/solver_bench.py ...
A=${A:-ab/lib_before.so}
for rep in 1 2; do
  echo "== A ($A) rep $rep"; MGT_LIB_PATH=$A "$@"
  echo "== B (in-tree) rep $rep"; "$@"
done
