# usage: bash tools/gpu_shapes.sh lib shape1 shape2 ...   (lib: variant name or "default")
v=$1; shift
if [ "$v" = default ]; then unset NTT_B200_LIB; else export NTT_B200_LIB=variants/libntt_$v.so; fi
for s in "$@"; do timeout 120 python tools/time_cfg.py $s 20 2>&1 | tail -1; done
