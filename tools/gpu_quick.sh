# quick GPU check: the GPU tests, then short bench lines (args: configs, default c4 c2 c3)
O=gpurun_out/${OUT:-quick}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
for c in ${@:-c4 c2 c3}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$? $(python -c "import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print(round(d['value']/1e9,1),'Gbfly/s',round(d['ms_per_step'],4),'ms',d['kernel_ms_mean'])" 2>&1 | tail -1)"
done
