cd $GRAFT_REPO_ROOT
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('value %.4e e2e %.4e frac %.3f evalfrac %.3f ms/step %.0f cpu %s'%(d['value'],d['e2e']['value'],d['roofline']['frac'],d['roofline']['dominant_kernel']['frac'],d['ms_per_step'],d['cpu_baseline']))"
