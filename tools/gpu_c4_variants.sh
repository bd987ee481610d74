# C4 A/B: the forward twiddle matrix and the column-pass tile order
O=gpurun_out/${OUT:-c4var}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
run() { # name env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --config ${CFG:-c4} --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$name.json 2> $O/bench_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('$O/bench_$name.json').read().strip().splitlines()[-1]);print(round(d['value']/1e9,1),'Gbfly/s',round(d['ms_per_step'],4),'ms',d['kernel_ms_mean'])" 2>&1 | tail -1)"
}
run base NTT_FS_MATRIX_MAX=0
run mat_cgi2 NTT_COLS_CGI=2
run mat_cgi0 NTT_COLS_CGI=0
run mat_cgi4 NTT_COLS_CGI=4
run mat_cgi6 NTT_COLS_CGI=6
run mat_nobm NTT_COLS_BMAJOR=0
run base2 NTT_FS_MATRIX_MAX=0
run mat_cgi2b NTT_COLS_CGI=2
