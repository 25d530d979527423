set -x
export PIFCM_E2E_OUT=gpurun_out/e2e_c3_r02.json
timeout 1500 python -m pytest tests/test_gpu_c3_e2e.py -x -q -s > gpurun_out/e2e.log 2>&1; tail -5 gpurun_out/e2e.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_stencil -s 1 -c 1 \
    -f -o gpurun_out/kstep_r02a python tools/profile_step.py eval 2 > gpurun_out/ncu_full_r02a.log 2>&1
tail -2 gpurun_out/ncu_full_r02a.log
TOOLS=initcheck bash tools/sanitize.sh
