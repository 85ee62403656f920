# GPU job: 24-bit split products in the packed plane MAC -- tests + A/B bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 1 0; do
HCNN_OPTIONS=mac_split=$v timeout 900 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_mac24_$v.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_mac24_$v.log').read().strip().splitlines()[-1])
print($v, d['ms_per_step'], d['logits_check'], {k:(v['share'],v['ms_per_launch'],v['launches'],v['GBps']) for k,v in list(d['kernels'].items())[:4]})"
done
