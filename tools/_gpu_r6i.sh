# permute gather: prefetching variant (MOE_B200_GATHER=pf) vs the default, standalone and
# in-step (alternating), plus the parity tests on the pf variant
for v in default pf default pf; do
  if [ $v = pf ]; then export MOE_B200_GATHER=pf; else unset MOE_B200_GATHER; fi
  timeout 200 python tools/hbm_probe.py 20 2>&1 | grep permute_gather | sed "s/^/[$v] /"
done
for c in qwen3 mixtral deepseek; do
for v in default pf default pf; do
  if [ $v = pf ]; then export MOE_B200_GATHER=pf; else unset MOE_B200_GATHER; fi
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-dropin > gpurun_out/r6i_$c_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r6i_$c_$v.json').read().strip().splitlines()[-1]);h=d['hbm_kernels']['moe_permute_gather'];print('[$v] $c', d['value'], d['ms_per_step'], h['ms_per_step'], h['frac_of_measured_hbm'])"
done
done
export MOE_B200_GATHER=pf
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_layer_scale_gpu.py tests/test_routing_api_gpu.py tests/test_ep_loopback_gpu.py -q -x -p no:cacheprovider > gpurun_out/r6i_pytest_pf.log 2>&1; tail -2 gpurun_out/r6i_pytest_pf.log
