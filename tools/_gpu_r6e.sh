# bench at N=2 with the union GEMM time / floor model (EP path), Mixtral + DeepSeek
for c in mixtral deepseek; do
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 2 --config $c > gpurun_out/r6e_bench2_$c.json 2> gpurun_out/r6e_bench2_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/r6e_bench2_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c', d['value'], d['ms_per_step'], r['bound'], r['frac'], r['gemm_ms_per_step'], r['floor_model']['frac_of_floor'], d['e2e']['value'])" || tail -5 gpurun_out/r6e_bench2_$c.err
done
