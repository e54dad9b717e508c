for spec in "base|_ab/lib_notma.so|" "l2|_ab/lib_notma.so|VOXSCHUR_DBG=512" "l3|_ab/lib_notma.so|VOXSCHUR_DBG=768" "l4|_ab/lib_notma.so|VOXSCHUR_DBG=1024" "l3p2|_ab/lib_notma.so|VOXSCHUR_DBG=800" "l3p2h2|_ab/lib_notma.so|VOXSCHUR_DBG=8992" "tma6|_ab/lib_tma6.so|" "tma8|_ab/lib_tma8.so|"; do
  IFS='|' read -r label lib envs <<< "$spec"
  echo "== $label"
  env $envs VOXSCHUR_CG=7 VOXSCHUR_X_DEPTH=4 VOXSCHUR_LIB=$(realpath $lib) timeout 200 python tools/prof_inner.py C4 1 2>&1 | grep -E "solve|phases|Error" | tail -4
done
