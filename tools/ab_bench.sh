# A/B of library variants on the C3 bench line: bash tools/ab_bench.sh lib1 lib2 ...
for rep in 1 2; do
for lib in "$@"; do
  PIFCM_LIB=$lib python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', round(d['value']/1e9,2), 'G', round(d['ms_per_step'],2), 'ms batched', round(r['avg_launch_ms']*1e3,1), 'us single', round(r['single_state_launches']['avg_launch_ms']*1e3,1), 'us', d['clocks']['sm_mhz'])"
done
done
