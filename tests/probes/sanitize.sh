# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the smoke workload and a
# small EEMD + CEEMDAN + serial/slicewise run (tests/probes/sanitize_work.py).
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 python tests/probes/sanitize_work.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.log >> gpurun_out/san/summary.txt
done
cat gpurun_out/san/summary.txt
