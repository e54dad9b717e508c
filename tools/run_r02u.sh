timeout 300 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02u_bench_c1.json 2> gpurun_out/r02u_c1.err; python - <<'P'
import json
b=json.load(open('gpurun_out/r02u_bench_c1.json'))
print('C1 ms/step', b['ms_per_step'], 'value', b['value'], [ (s['prec'], s['sms'], round(s['device_ms'],1)) for s in b['solves']], {k:round(v['us_per_cg_iteration'],1) for k,v in b['roofline']['kernels'].items()})
P
export VOXSCHUR_INNER_MAXIT=100
timeout 1200 python tools/ab_variants.py C4L "base:VOXSCHUR_CG=3" "mq:" --phases --rounds 1 > gpurun_out/r02u_ab_c4l.log 2>&1; cat gpurun_out/r02u_ab_c4l.log | cut -c1-330
