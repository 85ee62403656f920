# GPU job: chunk-pass register cap (ntt_occupancy=2) A/B, new lazy-MAC stress test, single-bootstrap breakdown
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for opt in "ntt_occupancy=0" "ntt_occupancy=2"; do
HCNN_OPTIONS=$opt python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_$opt.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_$opt.log').read().strip().splitlines()[-1])
print('$opt', d['ms_per_step'], d['roofline']['frac'], {k:(v['share'],v['ms_per_launch']) for k,v in list(d['kernels'].items())[:10]})"
done
timeout 600 python tools/boot_phases.py 1 2 2>&1 | tail -1
