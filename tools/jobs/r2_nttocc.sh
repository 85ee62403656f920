# GPU job: NTT occupancy / grouping knobs after the FP64 change
set -x
timeout 900 python tools/ntt_bench.py 0,1,0 0,1,1 64,1,0 128,1,0 2>&1 | grep limbs
for opt in "ntt_occupancy=1" "ntt_group_limbs=128"; do
HCNN_OPTIONS=$opt python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_$opt.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_$opt.log').read().strip().splitlines()[-1])
print('$opt', d['ms_per_step'], d['roofline']['frac'], {k:(v['share'],v['ms_per_launch']) for k,v in list(d['kernels'].items())[:8]})"
done
