#!/bin/bash
# same-box A/B of library builds: tools/ab.sh CONFIG lib1.so lib2.so ... (2 rounds each, alternating)
cfg=$1; shift
for round in 1 2; do
  for lib in "$@"; do
    echo "== $lib round $round"
    VOXSCHUR_LIB=$(realpath $lib) python tools/prof_inner.py $cfg 1 --no-phases | grep solve
  done
done
