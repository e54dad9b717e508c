VOXSCHUR_CG=6 VOXSCHUR_DBG=48 VOXSCHUR_INNER_MAXIT=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcgm" -c 1 \
  -o gpurun_out/r02p_c4_tile python tools/one_solve.py C4 1e-12 S > gpurun_out/r02p_ncu.log 2>&1
tail -3 gpurun_out/r02p_ncu.log
python tools/ncu_summary.py gpurun_out/r02p_c4_tile.ncu-rep 25 > gpurun_out/r02p_c4_tile.txt 2>&1; head -45 gpurun_out/r02p_c4_tile.txt
ncu -i gpurun_out/r02p_c4_tile.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k in ['l1tex__t_sector_hit_rate.pct','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum','lts__t_sectors_srcunit_tex_op_read.sum','lts__t_sectors_srcunit_tex_op_write.sum','lts__t_sector_hit_rate.pct','lts__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_elapsed','dram__throughput.avg.pct_of_peak_sustained_elapsed']:
    if k in h: print(k, v[h.index(k)])
"
