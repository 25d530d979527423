# One GPU call for a kernel change: parity of the step kernels with the
# default library, A/B device time of the fused step against variant
# libraries, and (NCU=1) a full ncu capture of the P = 32 launch with the
# per-instruction SASS counts.  Outputs in gpurun_out/.
#   bash tools/gpu_ab.sh lib_variant1.so lib_variant2.so ...
set -x
TAG=${TAG:-ab}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_step.py} -m gpu -q -x > gpurun_out/tests_${TAG}.log 2>&1
tail -5 gpurun_out/tests_${TAG}.log
bash tools/ab_time.sh paper_2002_01981_b200/libpifcm.so "$@" 2>&1 | tee gpurun_out/ab_${TAG}.txt
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_stencil -s 1 -c 1 \
      -f -o gpurun_out/kstep_${TAG} python tools/profile_step.py eval 2 > gpurun_out/ncu_${TAG}.log 2>&1
  tail -2 gpurun_out/ncu_${TAG}.log
  ncu -i gpurun_out/kstep_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}.csv 2>&1
  ncu -i gpurun_out/kstep_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}.csv 2>&1
  ls -la gpurun_out/
fi
