set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s3_pytest.log
timeout 300 python bench.py > gpurun_out/s3_bench_c4.json 2> gpurun_out/s3_bench_c4.err; echo "bench rc=$?"
timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/s3_bench_c3.json 2> gpurun_out/s3_bench_c3.err; echo "bench c3 rc=$?"
OUT=s3_prof bash tools/gpu_prof_src.sh
