# Round evidence: GPU tests, smoke, bench lines for every config, the ncu launch list of the
# default bench command and one ncu --set full capture of the top C2 kernels.
set -x
mkdir -p gpurun_out/ev
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1
for c in c2 c1 c3 c4 c5; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/ev/bench_$c.json 2> gpurun_out/ev/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_c2_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_c3_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_c4_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contig_tma -s 2 -c 2 -o gpurun_out/ev/prof_c2 python tools/prof_run.py c2 2 > gpurun_out/ev/ncu_c2_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_splitk|k_cols_tma" -c 3 -o gpurun_out/ev/prof_c4 python tools/prof_run.py c4 1 > gpurun_out/ev/ncu_c4_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_splitk" -c 3 -o gpurun_out/ev/prof_c3 python tools/prof_run.py c3 1 > gpurun_out/ev/ncu_c3_full.log 2>&1
ls -la gpurun_out/ev
