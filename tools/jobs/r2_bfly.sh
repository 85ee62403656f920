# GPU job: ncu of the butterfly-peak probe and of one NTT pair (instruction mix / pipes)
set -x
timeout 300 ncu --set full --clock-control none -k regex:"bfly_peak" -c 2 -o gpurun_out/bfly python -c "
import sys; sys.path.insert(0,'.')
from paper_2310_16530_b200 import _native
print(_native.ntt_butterfly_peak(True)/1e9, _native.ntt_butterfly_peak(False)/1e9)" > gpurun_out/ncu_bfly.log 2>&1; tail -2 gpurun_out/ncu_bfly.log
python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_kstma2.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_kstma2.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], {k:(v['share'],v['ms_per_launch'],v['GBps']) for k,v in list(d['kernels'].items())[:4]})"
