# GPU job: ks_inner variants (bit-identity + time), ncu of ks_inner / mac_multi in a ResNet20 image
set -x
timeout 900 python tools/ks_bench.py 0 2 3 4 > gpurun_out/ks_bench.log 2>&1; cat gpurun_out/ks_bench.log | grep -v "^$" | tail -40
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ks_inner|k_mac_multi" -s 200 -c 6 -o gpurun_out/r20_ks_mac python tools/r20_once.py > gpurun_out/ncu_ks.log 2>&1; tail -3 gpurun_out/ncu_ks.log
