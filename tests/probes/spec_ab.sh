# Speculative last sifts: GPU parity suite, then C5/C4 span probes with speculation on / off.
cd $GRAFT_REPO_ROOT
O=gpurun_out/spec
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${TESTS:-} > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -5 $O/pytest.log
for i in 1 2; do
  for sp in 1 0; do
    echo "== SEMD_SPEC=$sp"; SEMD_SPEC=$sp timeout 600 python tests/probes/gpu_probe17.py ${CFG:-c5} ${NR:-62} | tail -3
  done
done 2>&1 | tee $O/probe17.txt
