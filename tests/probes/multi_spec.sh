# Span probe over prebuilt library variants (libsemd_b200_<tag>.so), speculation on and off.
cd $GRAFT_REPO_ROOT
for i in 1 2; do
for tag in ${TAGS}; do
  for sp in ${SPECS:-1 0}; do
    echo "== $tag SEMD_SPEC=$sp"
    SEMD_SPEC=$sp SEMD_LIB=$PWD/paper_2106_15319_b200/libsemd_b200_$tag.so timeout 600 python tests/probes/gpu_probe17.py ${CFG:-c5} ${NR:-62} | tail -3
  done
done
done
