# GPU job: TMA ring depth A/B
set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "mac or rot or hmult" 2>&1 | tail -2
for opt in "tma_stages=4" "tma_stages=6" "tma_stages=8"; do
HCNN_OPTIONS=$opt python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_$opt.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_$opt.log').read().strip().splitlines()[-1])
print('$opt', d['ms_per_step'], {k:(v['share'],v['ms_per_launch'],v['GBps']) for k,v in list(d['kernels'].items())[:4]})"
done
