timeout 300 python -m pytest tests -q -m gpu -x -k "supplementary" > gpurun_out/r02d_tests.log 2>&1; tail -5 gpurun_out/r02d_tests.log | cut -c1-300
export VOXSCHUR_INNER_MAXIT=300
timeout 900 python tools/ab_variants.py C4 "mq:VOXSCHUR_CG=4" "mq_nogather:VOXSCHUR_CG=4,VOXSCHUR_DBG=1" "mq_pf2:VOXSCHUR_CG=4,VOXSCHUR_PREFETCH=2" "mq_pf0:VOXSCHUR_CG=4,VOXSCHUR_PREFETCH=0" "rc_nogather:VOXSCHUR_CG=5,VOXSCHUR_DBG=1" --phases --ops S --rounds 1 > gpurun_out/r02d_ab_c4.log 2>&1; cat gpurun_out/r02d_ab_c4.log | cut -c1-330
unset VOXSCHUR_INNER_MAXIT
VOXSCHUR_CG=4 VOXSCHUR_INNER_MAXIT=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcgm" -c 1 \
  -o gpurun_out/r02d_c4_mq python tools/one_solve.py C4 1e-12 S > gpurun_out/r02d_ncu.log 2>&1
tail -3 gpurun_out/r02d_ncu.log
python tools/ncu_summary.py gpurun_out/r02d_c4_mq.ncu-rep 40 > gpurun_out/r02d_c4_mq.txt 2>&1; head -70 gpurun_out/r02d_c4_mq.txt
