bash tools/ab_time.sh paper_2002_01981_b200/libpifcm.so paper_2002_01981_b200/libpifcm_fold.so
for lib in libpifcm.so libpifcm_fold.so; do
  PIFCM_LIB=paper_2002_01981_b200/$lib python bench.py --workload C2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib C2', round(d['ms_per_step'],3), 'batched', round(r['avg_launch_ms']*1e3,1), 'us single', round(r['single_state_launches']['avg_launch_ms']*1e3,1), 'us')"
done
PIFCM_LIB=paper_2002_01981_b200/libpifcm_fold.so python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
python bench.py --workload C4 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | tail -c 1200
