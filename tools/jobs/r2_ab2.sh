# GPU job: new launch shapes as defaults (128-thread plane MAC + key-switch inner product): full gpu tests,
# smoke, default bench line, and the previous shapes on the same box for A/B
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_v12.log 2>&1
HCNN_OPTIONS=mac_tpb=256,tma_stages=4,ks_tpb=256 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ab2_old.log 2>&1
for f in gpurun_out/bench_v12.log gpurun_out/ab2_old.log; do
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);k=d['kernels'];print(sys.argv[1],round(d['ms_per_step'],2),d['e2e']['value'],d['clocks'],k['mac_multi']['ms_per_launch'],k['ks_inner']['ms_per_launch'])" $f
done
