# GPU parity (fast subset unless FULL=1) + C5 step anatomy + C4 bench line.
cd $GRAFT_REPO_ROOT
if [ "${FULL:-0}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
else
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_comm.py -m gpu -x -q -p no:cacheprovider -k "not c4_full and not c5" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
fi
tail -3 gpurun_out/pytest_gpu.log
python tests/probes/gpu_probe17.py c5 62 2>&1 | tail -2
python tests/probes/gpu_probe17.py c4 100 2>&1 | tail -2
