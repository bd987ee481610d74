# usage: bash tools/gpu_sweep.sh CONFIG lib1 lib2 ...   (libs under variants/, "default" = in-tree)
cfg=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then unset NTT_B200_LIB; else export NTT_B200_LIB=variants/libntt_$v.so; fi
  timeout 120 python tools/time_cfg.py $cfg 20 2>&1 | tail -1
done
