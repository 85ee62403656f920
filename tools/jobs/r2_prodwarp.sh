# GPU job: producer-warp TMA kernels (full/empty mbarrier rings) -- parity + bench + stage depth
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/ks_bench.py "ks_tma=0,ks_pipe=2" "ks_tma=1" 2>&1 | grep case | grep -v nb1
for opt in "tma_stages=4" "tma_stages=6"; do
HCNN_OPTIONS=$opt python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_pw_$opt.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_pw_$opt.log').read().strip().splitlines()[-1])
print('$opt', d['ms_per_step'], {k:(v['share'],v['ms_per_launch'],v['GBps']) for k,v in list(d['kernels'].items())[:4]})"
done
