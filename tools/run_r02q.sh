timeout 600 python tools/ab_variants.py C3s32 "mq:VOXSCHUR_CG=4" "tq:VOXSCHUR_CG=6,VOXSCHUR_DBG=48" "tr:VOXSCHUR_CG=7,VOXSCHUR_DBG=48" "rc:VOXSCHUR_CG=5" --phases --rounds 1 --ops S > gpurun_out/r02q_ab_c3.log 2>&1; cat gpurun_out/r02q_ab_c3.log | cut -c1-330
for v in 4 6; do
VOXSCHUR_CG=$v VOXSCHUR_DBG=48 VOXSCHUR_INNER_MAXIT=60 timeout 600 ncu --metrics lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,dram__bytes_read.sum --clock-control none -k regex:"k_pcgm" -c 1 python tools/one_solve.py C3s32 1e-12 S 2>&1 | grep -E "lts__|gpu__time|l1tex|dram__|k_pcgm"
done
