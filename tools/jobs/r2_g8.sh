# GPU job: 8 outputs per shared-term MAC launch -- tests + bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_g8.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_g8.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['logits_check'], {k:(v['share'],v['ms_per_launch'],v['launches'],v['GBps']) for k,v in list(d['kernels'].items())[:6]})"
