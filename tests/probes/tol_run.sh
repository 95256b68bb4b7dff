# Tolerance-mode spline experiment: golden realizations, speed, and the whole C5 ensemble against the exact library.
cd $GRAFT_REPO_ROOT
O=gpurun_out/tol
mkdir -p $O
T=$PWD/paper_2106_15319_b200/libsemd_b200_tol.so
SEMD_LIB=$T python tests/probes/tol_experiment.py real c4 > $O/real_c4.txt 2>&1; tail -4 $O/real_c4.txt
SEMD_LIB=$T python tests/probes/tol_experiment.py real c5 > $O/real_c5.txt 2>&1; tail -6 $O/real_c5.txt
for i in 1 2; do
  echo "== exact"; python tests/probes/gpu_probe17.py c5 62 | tail -3 | head -2
  echo "== tol"; SEMD_LIB=$T python tests/probes/gpu_probe17.py c5 62 | tail -3 | head -2
done > $O/probe17.txt 2>&1; cat $O/probe17.txt
python tests/probes/tol_experiment.py dump c5 /tmp/c5_exact > $O/dump_exact.txt 2>&1; tail -1 $O/dump_exact.txt
SEMD_LIB=$T python tests/probes/tol_experiment.py dump c5 /tmp/c5_tol > $O/dump_tol.txt 2>&1; tail -1 $O/dump_tol.txt
python tests/probes/tol_experiment.py cmp /tmp/c5_exact /tmp/c5_tol > $O/cmp_c5.txt 2>&1; cat $O/cmp_c5.txt
