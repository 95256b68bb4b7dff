# Round-2 (second session) measurement set on the GPU box. Outputs under gpurun_out/r02b.
# Bench lines (C5 with its CPU baseline and the reference arm, C4, C3, C2), the C5 launch list,
# and ncu --set full captures of the dominant kernels: k_eval / k_solve / k_final on C5 and the
# resident engine's k_res_ceemdan (C3) and k_resident (C2).
cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
O=gpurun_out/${OUT:-r02c}
mkdir -p $O
timeout 1200 python bench.py > $O/bench_c5_n1.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_c5_reference.json 2> $O/bench_c5_ref.err; echo "ref c5 rc=$?"
timeout 600 python bench.py --config c4 --no-cpu > $O/bench_c4_n1.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 600 python bench.py --config c3 --steps 10 --e2e-steps 3 > $O/bench_c3_n1.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config c2 --steps 10 --e2e-steps 3 > $O/bench_c2_n1.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c3 --impl reference --steps 2 --warmup 1 > $O/bench_c3_reference.json 2> $O/bench_c3_ref.err
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu > $O/ncu_launches.log 2>&1
python tests/probes/ncu_summary.py $O/launches_c5.csv > $O/launches_c5_summary.txt 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
    python bench.py --config c3 --steps 1 --warmup 0 --no-cpu > $O/ncu_launches_c3.log 2>&1
python tests/probes/ncu_summary.py $O/launches_c3.csv > $O/launches_c3_summary.txt 2>&1
for spec in "c5 k_eval 12 eval_c5" "c5 k_solve 2 solve_c5" "c5 k_final 4 final_c5" "c5 k_eval 13 evalspec_c5" "c3 k_res_ceemdan 0 resident_c3" "c2 k_resident 0 resident_c2"; do
  set -- $spec
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:$2 -s $3 -c 1 \
      -o $O/$4 -f python bench.py --config $1 --steps 1 --warmup 0 --no-cpu > $O/ncu_$4.log 2>&1
  python tests/probes/ncu_extract.py $O/$4.ncu-rep $4 > $O/$4_summary.json 2>&1
done
ls -la $O
