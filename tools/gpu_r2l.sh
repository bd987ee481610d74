OUT=r2l bash tools/gpu_ab.sh "c3" splitnx2
O=gpurun_out/r2l
for cgi in 1 3 2; do
  NTT_COLS_CGI=$cgi timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $O/cgi$cgi.json 2>/dev/null
  echo "cgi=$cgi $(python -c "import json;d=json.loads(open('$O/cgi$cgi.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'ms',d['kernel_ms_mean'])")"
done
