# Round-2 evidence on one B200: GPU tests, smoke, the driver's default bench line (C4) and reference arm,
# the other configs' lines, the launch list of the default bench command, Table-1 per config.
O=gpurun_out/ev2
rm -rf $O && mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --impl reference > $O/ref_default.json 2> $O/ref_default.err; echo "reference rc=$?"
for c in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 python tools/table1_b200.py > $O/table1.json 2> $O/table1.err; echo "table1 rc=$?"
ls -la $O
# one ncu --set full capture of C4's two kernels (one launch each) for the summary and the traffic figures
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_splitk|k_cols_tma" -s 2 -c 2 \
  -o $O/c4_full python tools/prof_run.py c4 2 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/c4_full.ncu-rep --page raw --csv > $O/c4_full_raw.csv 2>/dev/null
