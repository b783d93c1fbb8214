# in-step wave-sync settings A/B (graph bench, Mixtral), two rounds
for i in 1 2; do
for v in "1 256 1 32" "0 256 1 32" "1 128 1 32" "1 256 2 32" "1 256 1 64"; do set -- $v
  MOE_B200_WAVE_SYNC=$1 MOE_B200_SYNC_MIN_KB=$2 MOE_B200_SYNC_LAG=$3 MOE_B200_SYNC_KB=$4 timeout 300 python bench.py --no-cpu-baseline --no-dropin --steps 30 > gpurun_out/r5p.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r5p.json').read().strip().splitlines()[-1]);print('sync=$1 min_kb=$2 lag=$3 kb=$4', d.get('ms_per_step'), 'mhz', (d.get('clocks') or {}).get('sm_mhz'))"
done
done
