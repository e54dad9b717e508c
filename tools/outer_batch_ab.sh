timeout 1300 python -m pytest tests -q -m gpu -x > gpurun_out/r02w_gpu_tests.log 2>&1; tail -4 gpurun_out/r02w_gpu_tests.log | cut -c1-300
for b in 1 4; do
VOXSCHUR_OUTER_BATCH=$b timeout 300 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu --sequential > gpurun_out/r02w_bench_c1_seq_batch$b.json 2> /dev/null
python - <<P
import json
b=json.load(open('gpurun_out/r02w_bench_c1_seq_batch$b.json'))
print('batch $b: C1 sequential ms/step', round(b['ms_per_step'],1), [ (s['prec'], s['iters_outer'], s['inner'], round(s['device_ms'],1), s['k']) for s in b['solves']])
P
done
timeout 300 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02w_bench_c1.json 2> /dev/null
timeout 300 python bench.py --config C0 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02w_bench_c0.json 2> /dev/null
python - <<P
import json
for f in ['c1','c0']:
    b=json.load(open('gpurun_out/r02w_bench_%s.json'%f))
    print(f, 'ms/step', round(b['ms_per_step'],1), 'value', round(b['value'],2), [ (s['prec'], s['sms'], round(s['device_ms'],1)) for s in b['solves']])
P
