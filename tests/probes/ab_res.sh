# A/B of a resident-engine change: per-phase cycles (probe 22) and C3/C2 bench step times for the
# working-tree library (A, at several SEMD_RES_CHAINS) and libsemd_b200_ab.so (B, HEAD's source),
# then the resident GPU tests on A.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab
mkdir -p $O
B=$PWD/paper_2106_15319_b200/libsemd_b200_ab.so
{
for i in 1 2; do
  echo "== B"; SEMD_LIB=$B python tests/probes/gpu_probe22.py c2 c3 2>&1 | tail -4
  for ch in ${CHAINS:-96 160 256}; do
    echo "== A chains $ch"; SEMD_RES_CHAINS=$ch python tests/probes/gpu_probe22.py c2 c3 2>&1 | tail -4
  done
done
for ch in ${CHAINS:-96 160 256}; do
  echo "== A bench c3 chains $ch"; SEMD_RES_CHAINS=$ch timeout 300 python bench.py --config c3 --steps 20 --e2e-steps 3 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3 ms/step %.3f e2e %.3e'%(d['ms_per_step'],d['e2e']['value']))"
done
echo "== B bench c3"; SEMD_LIB=$B timeout 300 python bench.py --config c3 --steps 20 --e2e-steps 3 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3 ms/step %.3f e2e %.3e'%(d['ms_per_step'],d['e2e']['value']))"
} > $O/res.txt 2>&1
cat $O/res.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${TESTS:-} > $O/pytest.log 2>&1; echo pytest_rc=$?
tail -3 $O/pytest.log
