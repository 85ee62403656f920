# GPU job: ncu --set full of the TMA-staged MAC and key-switch kernels inside a ResNet20 image
set -x
python tools/r20_once.py > gpurun_out/plain_r20.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mac_multi_tma" -s 40 -c 2 -o gpurun_out/r20_mac_tma python tools/r20_once.py > gpurun_out/ncu_mac_tma.log 2>&1; tail -1 gpurun_out/ncu_mac_tma.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ks_inner" -s 100 -c 4 -o gpurun_out/r20_ks_tma python tools/r20_once.py > gpurun_out/ncu_ks_tma.log 2>&1; tail -1 gpurun_out/ncu_ks_tma.log
