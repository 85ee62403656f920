# GPU job: routing threshold of the TMA key-switch inner product (batch entries) with the 128-thread kernel
set -x
for o in base ks_tma_min=2 ks_tma_min=1 base; do
  oo=$o; [ $o = base ] && oo=
  HCNN_OPTIONS=$oo timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ab3_$o.log 2>&1
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);k=d['kernels'];print(sys.argv[1],round(d['ms_per_step'],2),d['clocks']['reasons'],k['ks_inner'])" gpurun_out/ab3_$o.log
done
