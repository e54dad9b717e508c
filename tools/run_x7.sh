for spec in "nobpf|_ab/lib_nobpf.so|" "bpf|paper_2307_05266_b200/libvoxschur.so|" "bpf_p2|paper_2307_05266_b200/libvoxschur.so|VOXSCHUR_PREFETCH=2" "bpf_p3|paper_2307_05266_b200/libvoxschur.so|VOXSCHUR_PREFETCH=3" "wl2|_ab/lib_wl2.so|" "wl2nobpf|_ab/lib_wl2nobpf.so|" "wl2_p2|_ab/lib_wl2.so|VOXSCHUR_PREFETCH=2"; do
  IFS='|' read -r label lib envs <<< "$spec"
  echo "== $label"
  env $envs VOXSCHUR_CG=7 VOXSCHUR_X_DEPTH=4 VOXSCHUR_LIB=$(realpath $lib) timeout 200 python tools/prof_inner.py C4 1 2>&1 | grep -E "solve|phases|Error" | tail -4
done
