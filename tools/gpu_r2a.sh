# round-2 first GPU call: the GPU test suite, smoke, bench lines (C4 default, C2, C3, C5), launch list of C4
set -x
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
for c in c2 c3 c5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_c4.json 2> $O/ref_c4.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1; echo "ncu rc=$?"
