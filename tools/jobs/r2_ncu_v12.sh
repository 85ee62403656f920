# GPU job: ncu --set full of the 128-thread plane MAC / key-switch kernels (eager ResNet20 image),
# then the launch list of the timed bench step (v12 code)
set -x
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_mac_multi_tma2|k_ks_inner_tma2" -s 40 -c 4 \
  -o gpurun_out/r20_v12_tpb128 python tools/r20_once.py > gpurun_out/ncu_full_v12.log 2>&1
tail -2 gpurun_out/ncu_full_v12.log
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench_v12.log 2>&1 && \
timeout 2700 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_v12.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_v12.log 2>&1
tail -2 gpurun_out/ncu_launches_v12.log; wc -l gpurun_out/launches_v12.csv
