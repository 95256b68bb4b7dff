# Span probe over several prebuilt library variants (paper_2106_15319_b200/libsemd_b200_<tag>.so).
cd $GRAFT_REPO_ROOT
for tag in ${TAGS}; do
  echo "== $tag"
  SEMD_LIB=$PWD/paper_2106_15319_b200/libsemd_b200_$tag.so python tests/probes/gpu_probe17.py ${CFG:-c5} ${NR:-62} | tail -1
done
