#!/bin/bash
# Round-2 GPU evidence: parity tests, the C4 bench line, the ncu launch list of
# the bench command and one full ncu capture of its dominant kernels at C4.
# usage (on the GPU box): bash tools/round2_profile.sh TAG [skip-tests]
tag=${1:-r02}
mkdir -p gpurun_out
if [ -z "$2" ]; then
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${tag}_gpu_tests.log 2>&1; tail -5 gpurun_out/${tag}_gpu_tests.log
fi
timeout 1500 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_bench.json | cut -c1-3000
tail -3 gpurun_out/${tag}_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-extras \
  > gpurun_out/${tag}_ncu_list.log 2>&1
python tools/launch_share.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launch_list.txt 2>&1; head -30 gpurun_out/${tag}_launch_list.txt
VOXSCHUR_INNER_MAXIT=60 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_pcg" -c 2 \
  -o gpurun_out/${tag}_c4_full python tools/one_solve.py C4 1e-12 SA > gpurun_out/${tag}_ncu_full.log 2>&1
tail -4 gpurun_out/${tag}_ncu_full.log
python tools/ncu_summary.py gpurun_out/${tag}_c4_full.ncu-rep 14 > gpurun_out/${tag}_c4_full.txt 2>&1; head -40 gpurun_out/${tag}_c4_full.txt
