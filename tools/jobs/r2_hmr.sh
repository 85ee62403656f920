# GPU job: fused hmult+rescale in EvalMod -- tests + bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_hmr.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench_hmr.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['logits_check'], {k:(v['share'],v['ms_per_launch'],v['launches']) for k,v in list(d['kernels'].items())[:8]})"
timeout 600 python tools/boot16.py 2>&1 | tail -2
