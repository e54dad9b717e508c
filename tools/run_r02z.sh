timeout 600 python -m pytest tests -q -m gpu -x -k "blocked_kernel" > gpurun_out/r02z_tests.log 2>&1; tail -3 gpurun_out/r02z_tests.log | cut -c1-300
timeout 900 python tools/ab_variants.py C4 "mq:VOXSCHUR_CG=4" "blk:VOXSCHUR_CG=6" --phases --rounds 1 --ops S > gpurun_out/r02z_ab_c4.log 2>&1; cat gpurun_out/r02z_ab_c4.log | cut -c1-330
VOXSCHUR_CG=6 VOXSCHUR_INNER_MAXIT=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcgb" -c 1 \
  -o gpurun_out/r02z_c4_blk python tools/one_solve.py C4 1e-12 S > gpurun_out/r02z_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r02z_c4_blk.ncu-rep 30 > gpurun_out/r02z_c4_blk.txt 2>&1; head -50 gpurun_out/r02z_c4_blk.txt
