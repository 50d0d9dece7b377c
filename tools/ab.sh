#!/bin/bash
# Same-box A/B of kernel variants: tools/ab.sh "<bench cmd>" lib1.so lib2.so ...
# (each library built with tools/oz_bench.py --build-variant NAME CSRC_DIR);
# runs the command twice per library, interleaved, with CGL_LIB_OVERRIDE.
cmd="$1"; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib (rep $rep)"
    if [ "$lib" = default ]; then env -u CGL_LIB_OVERRIDE $cmd; else CGL_LIB_OVERRIDE=$lib $cmd; fi
  done
done
