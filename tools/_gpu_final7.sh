# Final bench lines with the 60-step default window (steady power state), all configs at
# N=1, the reference arm at its default, and smoke
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin7_smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/fin7_smoke.log; tail -2 gpurun_out/fin7_smoke.log
t0=$SECONDS; python bench.py > gpurun_out/fin7_bench1.json 2> gpurun_out/fin7_bench1.err; echo "bench wall $((SECONDS-t0)) s"
for c in qwen3 deepseek; do timeout 400 python bench.py --config $c > gpurun_out/fin7_bench1_$c.json 2> gpurun_out/fin7_bench1_$c.err; done
t0=$SECONDS; python bench.py --impl reference > gpurun_out/fin7_ref1.json 2> gpurun_out/fin7_ref1.err; echo "reference wall $((SECONDS-t0)) s"
for f in fin7_bench1 fin7_bench1_qwen3 fin7_bench1_deepseek fin7_ref1; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), d.get('steps'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('roofline') or {}).get('bound'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('gpu_launches'))"; done
