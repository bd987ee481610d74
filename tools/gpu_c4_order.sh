# C4 column-pass tile order / L2 promotion A/B (twiddle matrix)
O=gpurun_out/c4order
mkdir -p $O
run() { local name=$1; shift
  env "$@" timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $O/$name.json 2> $O/$name.err
  echo "$name $(python -c "import json;d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'ms',d['kernel_ms_mean'])" 2>&1 | tail -1)"
}
run bm1_cgi2
run bm2_cgi0 NTT_COLS_BMAJOR=2 NTT_COLS_CGI=0
run bm2_cgi1 NTT_COLS_BMAJOR=2 NTT_COLS_CGI=1
run bm2_cgi2 NTT_COLS_BMAJOR=2 NTT_COLS_CGI=2
run bm2_cgi0_p0 NTT_COLS_BMAJOR=2 NTT_COLS_CGI=0 NTT_COLS_L2PROMO=0
run bm2_cgi1_p128 NTT_COLS_BMAJOR=2 NTT_COLS_CGI=1 NTT_COLS_L2PROMO=128
run bm1_cgi2_p128 NTT_COLS_L2PROMO=128
run bm2_cgi3 NTT_COLS_BMAJOR=2 NTT_COLS_CGI=3
run bm1_cgi2b
