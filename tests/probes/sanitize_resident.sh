# compute-sanitizer (memcheck, racecheck, synccheck) over the resident-engine workload, then one
# small lockstep EMD with programmatic dependent launch off. Each run is time-boxed.
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
O=gpurun_out/san
mkdir -p $O
: > $O/summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 300 $CS --tool $tool --print-limit 20 python tests/probes/sanitize_resident.py > $O/resident_$tool.log 2>&1
  echo "resident $tool rc=$?" >> $O/summary.txt
  tail -2 $O/resident_$tool.log >> $O/summary.txt
done
SEMD_PDL=0 timeout 300 $CS --tool memcheck --print-limit 20 python tests/probes/sanitize_resident.py lockstep > $O/lockstep_memcheck.log 2>&1
echo "lockstep memcheck rc=$?" >> $O/summary.txt
tail -2 $O/lockstep_memcheck.log >> $O/summary.txt
cat $O/summary.txt
