# A/B of 2D step variants on C2 (bench.py --workload C2): bash tools/ab_2d.sh lib1 lib2 ...
for rep in 1 2; do
for lib in "$@"; do
  PIFCM_LIB=$lib python bench.py --workload C2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', round(d['ms_per_step'],3), 'batched', round(r['avg_launch_ms']*1e3,1), 'us single', round(r['single_state_launches']['avg_launch_ms']*1e3,1), 'us')"
done
done
