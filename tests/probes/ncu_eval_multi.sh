# ncu full captures of a few k_eval launches in a C5 wave (SKIP: first launch index, COUNT launches)
cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:${KERNEL:-k_eval} -s ${SKIP:-10} -c ${COUNT:-4} \
  -o gpurun_out/${OUT:-evalm} -f python tests/probes/gpu_probe6.py c5 31 > gpurun_out/${OUT:-evalm}.log 2>&1
ls -la gpurun_out/${OUT:-evalm}.ncu-rep
