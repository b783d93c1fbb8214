for i in 1 2 3; do
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin > gpurun_out/r2x_a$i.json 2>/dev/null
MOE_BENCH_KERNEL_EVENTS=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin > gpurun_out/r2x_b$i.json 2>/dev/null
done
for f in a1 b1 a2 b2 a3 b3; do python -c "
import json; d=json.load(open('gpurun_out/r2x_$f.json')); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['achieved'], d['clocks']['samples'])"; done
