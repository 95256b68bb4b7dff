# k_solve variants: HEAD (ab), shared slopes + reciprocal table (slope), + helper-warp value gather (help = the
# working tree). Span probe interleaved, the solve phase profile, the resident C3/C2 bench lines, then the GPU suite.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab3
mkdir -p $O
P=$PWD/paper_2106_15319_b200
for i in 1 2; do
  for tag in ${TAGS:-ab slope help}; do
    echo "== $tag"; SEMD_LIB=$P/libsemd_b200_$tag.so python tests/probes/gpu_probe17.py ${CFG:-c5} ${NR:-62} | tail -3 | head -2
  done
done > $O/probe17.txt 2>&1
cat $O/probe17.txt
for tag in ${TAGS:-ab slope help}; do
  echo "== $tag"; SEMD_LIB=$P/libsemd_b200_$tag.so python tests/probes/gpu_probe15.py c5 31 2>&1 | tail -12
done > $O/probe15.txt 2>&1
cat $O/probe15.txt
for tag in ab help; do
  echo "== $tag"; SEMD_LIB=$P/libsemd_b200_$tag.so python tests/probes/gpu_probe21.py c3 c2 2>&1 | tail -6
done > $O/probe21.txt 2>&1
cat $O/probe21.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -3 $O/pytest.log
