# GPU job: forward-only split default -- tests + full bench line
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench_v8.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_v8.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e'], d['roofline'], d['gpu_launches'], d['clocks'], {k:(v['share'],v['ms_per_launch']) for k,v in list(d['kernels'].items())[:8]})"
