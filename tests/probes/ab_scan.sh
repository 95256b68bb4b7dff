cd $GRAFT_REPO_ROOT
for lib in paper_2106_15319_b200/libsemd_b200.so paper_2106_15319_b200/libsemd_b200_b.so; do
  echo "== $lib"
  SEMD_LIB=$PWD/$lib python tests/probes/gpu_probe19.py c5 186 | tail -2
  SEMD_LIB=$PWD/$lib python tests/probes/gpu_probe19.py c4 100 | tail -2
done
