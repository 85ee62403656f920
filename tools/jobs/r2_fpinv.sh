# GPU job: FP64-quotient inverse NTT -- parity, NTT microbench, bench
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/ntt_bench.py 0,1,0,2 2>&1 | grep limbs
python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_fpinv.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_fpinv.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], {k:(v['share'],v['ms_per_launch']) for k,v in list(d['kernels'].items())[:14]})"
