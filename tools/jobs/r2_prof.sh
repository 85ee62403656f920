# GPU job: ncu --set full of the TMA MAC / key-switch kernels and the FP64 NTT in a ResNet20 image; bootstrap phases
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mac_multi_tma|k_ks_inner_tma|ntt2_fwd" -s 300 -c 8 -o gpurun_out/r20_v7 python tools/r20_once.py > gpurun_out/ncu_v7.log 2>&1; tail -2 gpurun_out/ncu_v7.log
timeout 600 python tools/boot_phases.py 2>&1 | tail -5
