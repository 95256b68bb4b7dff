# Wave-size sweep on C5: steps per wave and sifted samples/s vs SEMD_STEP_SAMPLES.
cd $GRAFT_REPO_ROOT
for s in 268435456 536870912 1073741824 2147483648; do
  echo "== SEMD_STEP_SAMPLES=$s"
  SEMD_STEP_SAMPLES=$s timeout 300 python tests/probes/gpu_probe6.py c5 ${NR:-120}
done
