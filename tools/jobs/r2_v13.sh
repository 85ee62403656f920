# GPU job: TMA inner product from 2 batch entries: full gpu tests, smoke, default bench line
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_v13.log 2>&1
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);k=d['kernels'];print(round(d['ms_per_step'],2),d['e2e']['value'],d['clocks'],k['ks_inner'])" gpurun_out/bench_v13.log
