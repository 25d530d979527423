timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_pso.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
bash tools/ab_time.sh paper_2002_01981_b200/libpifcm.so paper_2002_01981_b200/libv_sy0.so 2>&1
bash tools/ab_bench.sh paper_2002_01981_b200/libpifcm.so paper_2002_01981_b200/libv_sy0.so 2>&1
for lib in paper_2002_01981_b200/libpifcm.so paper_2002_01981_b200/libv_tyb2.so paper_2002_01981_b200/libv_tyb1.so; do
  PIFCM_LIB=$lib timeout 600 python bench.py --workload C2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib C2', round(d['ms_per_step'],3), 'ms batched', round(r['avg_launch_ms']*1e3,1), 'us single', round(r['single_state_launches']['avg_launch_ms']*1e3,1), 'us')"
done
