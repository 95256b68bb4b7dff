# GPU parity suite, then the default C5 bench (no CPU leg), for quick iteration.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('value %.4e e2e %.4e frac %.3f eval_ms %.0f ms/step %.0f'%(d['value'],d['e2e']['value'],d['roofline']['frac'],d['roofline']['dominant_kernel']['ms_per_step'],d['ms_per_step']))"
