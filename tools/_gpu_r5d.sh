# MXFP8 (all six expert GEMMs) bench line at the final state, next to bf16 on the same box
timeout 400 python bench.py --precision mxfp8 --no-cpu-baseline --no-dropin > gpurun_out/r5d_mx.json 2> gpurun_out/r5d_mx.err
timeout 400 python bench.py --no-cpu-baseline --no-dropin > gpurun_out/r5d_bf16.json 2> gpurun_out/r5d_bf16.err
for f in r5d_mx r5d_bf16; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'), d.get('dtype')[:20])"; done
tail -3 gpurun_out/r5d_mx.err
