# GPU job: TMA-staged plane MAC + ks_inner running pointers -- parity, bench, option A/B
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/ks_bench.py 2 2>&1 | grep case
for opt in "mac_tma=1" "mac_tma=0"; do
HCNN_OPTIONS=$opt python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_$opt.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_$opt.log').read().strip().splitlines()[-1])
print('$opt', d['ms_per_step'], d['roofline']['frac'], {k:(v['share'],v['ms_per_launch'],v['GBps']) for k,v in list(d['kernels'].items())[:6]})"
done
