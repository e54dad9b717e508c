#!/bin/bash
# tools/run_ab.sh CONFIG "label|lib.so|ENV=V ..." ...  -- one prof_inner run (with phase timers) per spec
cfg=$1; shift
for spec in "$@"; do
  IFS='|' read -r label lib envs <<< "$spec"
  echo "== $label"
  env $envs VOXSCHUR_LIB=$(realpath $lib) timeout 300 python tools/prof_inner.py $cfg 1 2>&1 | grep -E "solve|phases|Error" | tail -4
done
