# A/B of a k_solve change: solve phase profile (probe 15) and kernel spans (probe 17) for the
# working-tree library (A) and libsemd_b200_ab.so (B, HEAD's semd_sift.cu), then the GPU parity
# suite on A.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab
mkdir -p $O
B=$PWD/paper_2106_15319_b200/libsemd_b200_ab.so
for i in 1 2; do
  echo "== A"; python tests/probes/gpu_probe15.py c5 31 2>&1 | tail -12
  echo "== B"; SEMD_LIB=$B python tests/probes/gpu_probe15.py c5 31 2>&1 | tail -12
done > $O/probe15.txt
for i in 1 2; do
  echo "== A"; python tests/probes/gpu_probe17.py ${CFG:-c5} ${NR:-62} | tail -2
  echo "== B"; SEMD_LIB=$B python tests/probes/gpu_probe17.py ${CFG:-c5} ${NR:-62} | tail -2
done > $O/probe17.txt
cat $O/probe15.txt $O/probe17.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${TESTS:-} > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -3 $O/pytest.log
