set -x
timeout 600 python -m pytest tests/test_gpu_slab_pso.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 --cpu-budget 20 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -c 3000 gpurun_out/bench_c5.json; tail -5 gpurun_out/bench_c5.err
