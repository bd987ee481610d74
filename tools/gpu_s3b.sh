# session-3 A/B: GPU tests with the default library, then bench lines default vs abvar variants
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3b_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s3b_pytest.log
OUT=${ABOUT:-s3b_ab} bash tools/gpu_ab.sh "${ABCFG:-c4 c3}" "$@"
