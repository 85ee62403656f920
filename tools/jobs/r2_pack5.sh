# GPU job: 40/48-bit per-prime packed masks -- parity + bench
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_pack5.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_pack5.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['config']['resident_mask_gb'], d['setup'], d['logits_check'], {k:(v['share'],v['ms_per_launch'],v['launches']) for k,v in list(d['kernels'].items())[:10]})"
