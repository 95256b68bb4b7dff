set -x
cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k_eval -s 6 -c 1 -o gpurun_out/eval_full -f python tests/probes/gpu_probe6.py c5 15 > gpurun_out/ncu_eval.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k_solve -s 6 -c 1 -o gpurun_out/solve_full -f python tests/probes/gpu_probe6.py c5 15 > gpurun_out/ncu_solve.log 2>&1
