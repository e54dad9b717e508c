#!/bin/bash
# same-box A/B of library builds and env settings on one config's inner solves:
#   tools/ab_env.sh CONFIG "LABEL|lib.so|ENV=V ..." ...   (2 rounds, alternating)
cfg=$1; shift
for round in 1 2; do
  for spec in "$@"; do
    IFS='|' read -r label lib envs <<< "$spec"
    echo "== $label round $round"
    env $envs VOXSCHUR_LIB=$(realpath $lib) python tools/prof_inner.py $cfg 1 --no-phases | grep -- "-solve"
  done
done
