# ncu --set full captures of the split-kernel shapes (C3's u32 2^16 conv, C4's u64 2^15 row pass).
rm -rf gpurun_out/ps && mkdir -p gpurun_out/ps
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -c 3 -o gpurun_out/ps/c3 python tools/prof_run.py c3 1 > gpurun_out/ps/c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -s 2 -c 1 -o gpurun_out/ps/u64 python tools/time_cfg.py x:4179340454199820289:64:15:2048:fwd 1 > gpurun_out/ps/u64.log 2>&1
ls -la gpurun_out/ps
