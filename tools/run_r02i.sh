timeout 900 python tools/ab_variants.py C4 "mq:VOXSCHUR_CG=4" --phases --rounds 1 > gpurun_out/r02i_ab_c4.log 2>&1; cat gpurun_out/r02i_ab_c4.log | cut -c1-330
timeout 600 python tools/ab_variants.py C2 "mq:VOXSCHUR_CG=4" --phases --rounds 1 > gpurun_out/r02i_ab_c2.log 2>&1; cat gpurun_out/r02i_ab_c2.log | cut -c1-330
