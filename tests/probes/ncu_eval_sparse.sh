# ncu full captures of k_eval launches late in a C5 wave (sparse IMFs) and early (dense).
cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
for s in ${SKIPS:-3 40}; do
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k_eval -s $s -c 1 -o gpurun_out/eval_s$s -f python tests/probes/gpu_probe6.py c5 31 > gpurun_out/ncu_eval_s$s.log 2>&1
done
