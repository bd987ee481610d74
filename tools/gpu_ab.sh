# A/B of library variants: bench lines for the default library and each abvar/ variant, interleaved
# usage: bash tools/gpu_ab.sh "c4 c2" variant1 [variant2 ...]
O=gpurun_out/${OUT:-ab}
mkdir -p $O
cfgs=$1; shift
for rep in 1 2; do
  for v in default "$@"; do
    for c in $cfgs; do
      if [ $v = default ]; then lib=""; else lib=abvar/libntt_$v.so; fi
      NTT_B200_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/${v}_${c}_$rep.json 2> $O/${v}_${c}_$rep.err
      echo "$v $c #$rep $(python -c "import json;d=json.loads(open('$O/${v}_${c}_$rep.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'ms',d['kernel_ms_mean'])" 2>&1 | tail -1)"
    done
  done
done
