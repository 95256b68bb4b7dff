# Wave-size sweep (span probe) at NR=250 for 512M / 768M / 1G samples per step.
cd $GRAFT_REPO_ROOT
for s in 536870912 805306368 1073741824; do
  echo "== SEMD_STEP_SAMPLES=$s"
  SEMD_STEP_SAMPLES=$s python tests/probes/gpu_probe17.py c5 ${NR:-250} | grep -A1 wall | tail -2
done
