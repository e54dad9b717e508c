#!/bin/bash
# Round-end GPU evidence: parity tests, the bench line, the ncu launch list of
# the bench command and one full ncu capture of its dominant kernel.
# usage (on the GPU box): bash tools/round_profile.sh TAG
tag=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${tag}_gpu_tests.log 2>&1; tail -2 gpurun_out/${tag}_gpu_tests.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_bench.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-hbm \
  > gpurun_out/${tag}_ncu_list.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cg1|k_pcg" --launch-skip 300 -c 2 \
  -o gpurun_out/${tag}_full python bench.py --steps 1 --warmup 3 --no-cpu --no-hbm > gpurun_out/${tag}_ncu_full.log 2>&1
tail -2 gpurun_out/${tag}_ncu_full.log
