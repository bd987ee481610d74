O=gpurun_out/c5mat
mkdir -p $O
for v in 24 28 24 28; do
  NTT_FS_MATRIX_MAX=$v timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/m$v.json 2>$O/m$v.err
  echo "max=$v $(python -c "import json;d=json.loads(open('$O/m$v.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'ms',d['kernel_ms_mean'])" 2>&1 | tail -1)"
done
NTT_FS_MATRIX_MAX=28 timeout 900 python -m pytest tests -m gpu -x -q -k "config5 or three_pass or device_resident" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
