# Wave-size sweep (span probe) at NR=186: 320M / 384M / 512M samples per step.
cd $GRAFT_REPO_ROOT
for s in 335544320 402653184 536870912; do
  echo "== SEMD_STEP_SAMPLES=$s"
  SEMD_STEP_SAMPLES=$s python tests/probes/gpu_probe17.py c5 ${NR:-186} | grep -A1 wall | tail -2
done
