# Round evidence, part 1 (small outputs): GPU tests, smoke, bench lines for every config and the ncu
# launch lists of the bench commands.  Part 2 (tools/gpu_round_profiles.sh) captures ncu --set full.
set -x
rm -rf gpurun_out/ev && mkdir -p gpurun_out/ev
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1
for c in c2 c1 c3 c4 c5; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/ev/bench_$c.json 2> gpurun_out/ev/bench_$c.err; done
for c in c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_${c}_bench.log 2>&1
done
ls -la gpurun_out/ev
