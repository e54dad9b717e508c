# time to tolerance with clock records (bench.py samples nvidia-smi during the timed step)
# usage: bash tools/time_to_tol.sh TAG
tag=${1:-r02s}
timeout 300 python bench.py --config C2 --steps 2 --warmup 3 --no-cpu > gpurun_out/${tag}_bench_c2_to_tol.json 2> gpurun_out/${tag}_c2.err; cut -c1-900 gpurun_out/${tag}_bench_c2_to_tol.json
timeout 300 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu > gpurun_out/${tag}_bench_c1_to_tol.json 2> gpurun_out/${tag}_c1.err; cut -c1-600 gpurun_out/${tag}_bench_c1_to_tol.json
timeout 1500 python bench.py --config C4 --max-outer 1000 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${tag}_bench_c4_to_tol.json 2> gpurun_out/${tag}_c4.err; cut -c1-1500 gpurun_out/${tag}_bench_c4_to_tol.json
