O=gpurun_out/r2d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python tools/table1_b200.py > $O/table1.json 2> $O/table1.err; echo "table1 rc=$?"
for c in c4 c2 c3 c5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$? $(python -c "import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print(round(d['value']/1e9,1),'Gbfly/s',round(d['ms_per_step'],4),'ms',d['kernel_ms_mean'])" 2>&1 | tail -1)"
done
