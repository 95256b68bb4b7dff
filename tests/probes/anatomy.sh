# Step anatomy (per-kernel device spans) on C5/C4/C2 and the C3 bench line.
cd $GRAFT_REPO_ROOT
python tests/probes/gpu_probe17.py c5 62 > gpurun_out/anat_c5.log 2>&1
python tests/probes/gpu_probe17.py c4 100 > gpurun_out/anat_c4.log 2>&1
python tests/probes/gpu_probe17.py c2 100 > gpurun_out/anat_c2.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu --steps 5 --e2e-steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config c2 --no-cpu --steps 5 --e2e-steps 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -n 4 gpurun_out/anat_*.log
python -c "
import json
for c in ('c2','c3'):
    d=json.load(open('gpurun_out/bench_%s.json'%c));print(c,'value %.3e ms/step %.2f e2e %.3e'%(d['value'],d['ms_per_step'],d['e2e']['value']))"
