# A/B device time of the fused step (C3, P = 32, and the single-state
# canonical launches) for library variants: bash tools/ab_time.sh lib1 lib2 ...
for rep in 1 2; do
  for lib in "$@"; do
    echo "$lib: $(PIFCM_LIB=$lib python tools/profile_step.py time 2>&1 | grep -E 'fused step|single state' | tr '\n' ' ')"
  done
done
