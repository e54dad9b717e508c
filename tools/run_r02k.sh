timeout 900 python -m pytest tests -q -m gpu -x -k "pcgm_qrec or (other_kernels and 4) or (descriptor and 4) or C1_simple or C2_simple_cap1 or slit_known" > gpurun_out/r02k_tests.log 2>&1; tail -4 gpurun_out/r02k_tests.log | cut -c1-300
timeout 900 python tools/ab_variants.py C4 "mq:VOXSCHUR_CG=4" --phases --rounds 1 > gpurun_out/r02k_ab_c4.log 2>&1; cat gpurun_out/r02k_ab_c4.log | cut -c1-330
timeout 600 python tools/ab_variants.py C2 "mq:VOXSCHUR_CG=4" --phases --rounds 1 > gpurun_out/r02k_ab_c2.log 2>&1; cat gpurun_out/r02k_ab_c2.log | cut -c1-330
