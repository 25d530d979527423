for lib in libpifcm.so libpifcm_tyb8.so libpifcm_tyb2.so libpifcm_mb5.so; do
  PIFCM_LIB=paper_2002_01981_b200/$lib python bench.py --workload C2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', round(d['ms_per_step'],3), 'batched', round(r['avg_launch_ms']*1e3,1), 'us single', round(r['single_state_launches']['avg_launch_ms']*1e3,1), 'us')"
done
python -m pytest tests/test_gpu_pso.py tests/test_gpu_inputs.py tests/test_gpu_slab_pso.py tests/test_gpu_slice.py tests/test_gpu_dist.py -q -x 2>&1 | tail -3
python tools/profile_step.py segment >/dev/null 2>&1
