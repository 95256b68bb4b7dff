# Round-2 measurement set (GPU box). Outputs under gpurun_out/r02prof.
cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
O=gpurun_out/r02prof
mkdir -p $O
timeout 1200 python bench.py > $O/bench_c5_n1.json 2> $O/bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_c5_reference.json 2> $O/bench_c5_ref.err; echo "ref c5 rc=$?"
timeout 600 python bench.py --config c4 --no-cpu > $O/bench_c4_n1.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c3 --e2e-steps 3 > $O/bench_c3_n1.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c2 --e2e-steps 3 > $O/bench_c2_n1.json 2> $O/bench_c2.err
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu > $O/ncu_launches.log 2>&1
python tests/probes/ncu_summary.py $O/launches_c5.csv > $O/launches_c5_summary.txt 2>&1
for spec in "k_eval 12 eval_c5" "k_solve 12 solve_c5" "k_final 1 final_c5"; do
  set -- $spec
  timeout 900 $NCU --set full --import-source on --clock-control none -k regex:$1 -s $2 -c 1 \
      -o $O/$3 -f python bench.py --steps 1 --warmup 0 --no-cpu > $O/ncu_$3.log 2>&1
  python tests/probes/ncu_extract.py $O/$3.ncu-rep $3 > $O/$3_summary.json 2>&1
done
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_eval -s 12 -c 1 \
    -o $O/eval_c4 -f python bench.py --config c4 --steps 1 --warmup 0 --no-cpu > $O/ncu_eval_c4.log 2>&1
python tests/probes/ncu_extract.py $O/eval_c4.ncu-rep eval_c4 > $O/eval_c4_summary.json 2>&1
ls -la $O
