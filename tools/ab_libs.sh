#!/bin/bash
# same-box A/B of library builds (tools/build_variant.sh) on one config's inner solves, with phase timers:
#   tools/ab_libs.sh CONFIG "ENV=V ..." lib1.so lib2.so ...   (2 rounds, alternating)
cfg=$1; envs=$2; shift 2
for round in 1 2; do
  for lib in "$@"; do
    echo "== $(basename $lib) round $round"
    env $envs VOXSCHUR_LIB=$(realpath $lib) python tools/prof_inner.py $cfg 1 | grep -E "solve|phases"
  done
done
