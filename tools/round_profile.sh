# One GPU call: the GPU test suite, the bench line, the reference arm, the
# launch list of one bench step, a full ncu capture of the fused step kernel
# (P = 32 launch) with its per-instruction SASS page, the other configs'
# bench lines and compute-sanitizer on the stencil kernels.  Outputs in
# gpurun_out/ (summaries copied to profiles/ by hand).
set -x
TAG=${TAG:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$NOTESTS" ]; then
  PIFCM_E2E_OUT=gpurun_out/e2e_c3_${TAG}.json timeout 2400 python -m pytest tests -m gpu -q -rs \
      > gpurun_out/gputests_${TAG}.log 2>&1
  tail -5 gpurun_out/gputests_${TAG}.log
fi
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_${TAG}.log 2>&1
tail -2 gpurun_out/smoke_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -c 3000 gpurun_out/bench_${TAG}.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2>&1
tail -c 1500 gpurun_out/bench_ref_${TAG}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python tools/profile_step.py segment > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_stencil -s 1 -c 1 \
    -f -o gpurun_out/kstep_${TAG} python tools/profile_step.py eval 2 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}.log
ncu -i gpurun_out/kstep_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}.csv 2>&1
timeout 900 python bench.py --workload C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err
tail -c 1500 gpurun_out/bench_c5_${TAG}.json
timeout 600 python bench.py --workload C2 --steps 5 --warmup 3 > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err
tail -c 1500 gpurun_out/bench_c2_${TAG}.json
timeout 900 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_${TAG}.json 2> gpurun_out/bench_c4_${TAG}.err
tail -c 800 gpurun_out/bench_c4_${TAG}.json
# (compute-sanitizer is closed on the GPU pool; SAN=1 runs it where allowed)
[ -n "$SAN" ] && bash tools/sanitize.sh ${SANCASES:-3d v2 pipe modes}
[ -n "$SHELLS" ] && timeout 900 python tools/time_shells.py > gpurun_out/time_shells_${TAG}.json 2> gpurun_out/time_shells.err
# CPU only: the oracle against itself from an fp32-rounded start at C3 (DESIGN 7)
[ -n "$CHAOS" ] && timeout 2400 python tools/chaos_c3.py gpurun_out/chaos_c3_${TAG}.json > gpurun_out/chaos.log 2>&1
true
