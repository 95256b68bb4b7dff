# kSolveWarm sweep: span probe + solve phase profile per prebuilt variant (libsemd_b200_w<W>.so).
cd $GRAFT_REPO_ROOT
for w in base ${WARMS:-24 28}; do
  if [ $w = base ]; then lib=$PWD/paper_2106_15319_b200/libsemd_b200.so; else lib=$PWD/paper_2106_15319_b200/libsemd_b200_w$w.so; fi
  echo "== $w"
  SEMD_LIB=$lib python tests/probes/gpu_probe17.py c5 62 | tail -1
  SEMD_LIB=$lib python tests/probes/gpu_probe15.py c5 31 | grep -E "rounds|phase"
done
