# Round evidence, part 2: one ncu --set full capture per config's dominant kernels (run with the
# config as argument, one per gpurun call, so each report fits the copy-back limit).
c=$1
rm -rf gpurun_out/prof && mkdir -p gpurun_out/prof
case $c in
  c2) timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contig_tma -s 2 -c 2 -o gpurun_out/prof/prof_c2 python tools/prof_run.py c2 2 ;;
  c3) timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -c 3 -o gpurun_out/prof/prof_c3 python tools/prof_run.py c3 1 ;;
  c4) timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_splitk|k_cols_tma" -c 2 -o gpurun_out/prof/prof_c4 python tools/prof_run.py c4 1 ;;
  c5) timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma|k_contig_tma" -c 3 -o gpurun_out/prof/prof_c5 python tools/prof_run.py c5 1 ;;
esac > gpurun_out/prof/ncu_$c.log 2>&1
ls -la gpurun_out/prof
