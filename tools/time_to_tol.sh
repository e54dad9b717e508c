# time to tolerance with clock records (bench.py samples nvidia-smi during the timed step)
timeout 300 python bench.py --config C2 --steps 2 --warmup 3 --no-cpu > gpurun_out/r02s_bench_c2_to_tol.json 2> gpurun_out/r02s_c2.err; cut -c1-900 gpurun_out/r02s_bench_c2_to_tol.json
timeout 300 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02s_bench_c1_to_tol.json 2> gpurun_out/r02s_c1.err; cut -c1-600 gpurun_out/r02s_bench_c1_to_tol.json
timeout 1500 python bench.py --config C4 --max-outer 1000 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02s_bench_c4_to_tol.json 2> gpurun_out/r02s_c4.err; cut -c1-1500 gpurun_out/r02s_bench_c4_to_tol.json
