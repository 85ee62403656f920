# GPU job: launch-shape A/B (one box, one build): plane MAC / key-switch inner product threads per CTA
set -x
timeout 600 python -m pytest tests/test_gpu_small.py -m gpu -x -q 2>&1 | tail -1
for o in base mac_tpb=128,tma_stages=3 ks_tpb=128,ks_stages=3 mac_tpb=128,tma_stages=3,mac_minb=5 ks_tpb=128,ks_stages=4 base; do
  oo=$o; [ $o = base ] && oo=
  HCNN_OPTIONS=$oo timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ab_$o.log 2>&1
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);k=d['kernels'];print(sys.argv[1],round(d['ms_per_step'],2),d['clocks']['reasons'],k['mac_multi']['ms_per_launch'],k['ks_inner']['ms_per_launch'])" gpurun_out/ab_$o.log
done
