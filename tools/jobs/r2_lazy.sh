# GPU job: lazy-MAC kernels -- parity tests, ks_inner variants, bench
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/ks_bench.py 0 2 4 2>&1 | grep case
python bench.py > gpurun_out/bench3.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench3.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], {k:(v['share'],v['ms_per_launch'],v['GBps']) for k,v in list(d['kernels'].items())[:8]})"
