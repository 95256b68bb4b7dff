# Round-end measurement set (GPU box): C5 bench (with CPU legs), C4/C3 benches, the ncu launch
# list of the C5 bench command, and one ncu --set full capture of a SIFT-mode k_eval launch.
cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
O=gpurun_out/prof
mkdir -p $O
timeout 900 python bench.py > $O/bench_c5_n1.json 2> $O/bench_c5.err
timeout 600 python bench.py --config c4 --no-cpu > $O/bench_c4_n1.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c3 --e2e-steps 5 > $O/bench_c3_n1.json 2> $O/bench_c3.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_launches.log 2>&1
python tests/probes/ncu_summary.py $O/launches_c5.csv > $O/launches_c5_summary.txt 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_eval -s ${EVAL_SKIP:-12} -c 1 \
    -o $O/eval_full -f python bench.py --steps 1 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1
ls -la $O
