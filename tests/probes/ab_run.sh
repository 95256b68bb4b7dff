# A/B: working-tree library (A) vs libsemd_b200_ab.so (B) on the span probe, interleaved.
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  echo A; python tests/probes/gpu_probe17.py ${CFG:-c5} ${NR:-62} | tail -1
  echo B; SEMD_LIB=$PWD/paper_2106_15319_b200/libsemd_b200_ab.so python tests/probes/gpu_probe17.py ${CFG:-c5} ${NR:-62} | tail -1
done
