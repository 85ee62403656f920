# GPU job: per-class NTT launches (split) vs run-time class selection
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
HCNN_OPTIONS=ntt_split=1 timeout 600 python -m pytest tests -m gpu -x -q -k "ntt or hmult or rot or resc" 2>&1 | tail -2
timeout 900 python tools/ntt_bench.py 0,1,0,0 0,1,0,1 2>&1 | grep limbs
for opt in "ntt_split=0" "ntt_split=1"; do
HCNN_OPTIONS=$opt python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_$opt.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_$opt.log').read().strip().splitlines()[-1])
print('$opt', d['ms_per_step'], d['roofline']['frac'], {k:(v['share'],v['ms_per_launch']) for k,v in list(d['kernels'].items())[:8]})"
done
