# A/B of library variants through tools/time_cfg.py (per-op medians, L2 flushed), interleaved, 2 reps
# usage: bash tools/gpu_ab_time.sh "c3 x:4179340454199820289:64:15:2048:inv" variant1 [variant2 ...]
O=gpurun_out/${OUT:-abt}
mkdir -p $O
cfgs=$1; shift
for rep in 1 2; do
  for v in default "$@"; do
    for c in $cfgs; do
      if [ $v = default ]; then lib=""; else lib=abvar/libntt_$v.so; fi
      echo "$v #$rep $(NTT_B200_LIB=$lib timeout 300 python tools/time_cfg.py $c 20 2>&1 | tail -n 1)"
    done
  done
done
