# Sustained A/B of library variants: the C3 bench line (power-capped clocks
# included) and the DRAM bytes of one P = 32 launch (ncu) per library.
#   bash tools/ab_bench.sh lib1.so lib2.so ...
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    PIFCM_LIB=$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', round(d['value']/1e9,2), 'G vp/s', round(d['ms_per_step'],2), 'ms/step launch', round(r['avg_launch_ms'],4), 'clk', d['clocks']['sm_mhz'])"
  done
done
for lib in "$@"; do
  PIFCM_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_step_stencil -s 1 -c 1 python tools/profile_step.py eval 2 2>/dev/null | grep -E "dram__bytes|duration" | sed "s|^|$lib |"
done
