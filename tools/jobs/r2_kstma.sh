# GPU job: TMA-staged key-switch inner product -- parity, A/B, bench
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/ks_bench.py "ks_tma=0,ks_pipe=2" "ks_tma=1" 2>&1 | grep case
python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_kstma.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_kstma.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], {k:(v['share'],v['ms_per_launch'],v['GBps']) for k,v in list(d['kernels'].items())[:10]})"
