# GPU job: plane MAC threads-per-CTA x register-cap sweep (bit-exactness + ResNet20 ms/image)
set -x
for o in mac_tpb=128,tma_stages=3,mac_minb=5 mac_tpb=128,tma_stages=2 mac_tpb=256,mac_minb=4; do
  HCNN_OPTIONS=$o timeout 600 python -m pytest tests/test_gpu_small.py tests/test_gpu_layers.py tests/test_gpu_hashes.py -m gpu -x -q 2>&1 | tail -1
done
for o in mac_tpb=128,tma_stages=3 mac_tpb=128,tma_stages=3,mac_minb=4 mac_tpb=128,tma_stages=3,mac_minb=5 mac_tpb=128,tma_stages=2 mac_tpb=256,mac_minb=4; do
  HCNN_OPTIONS=$o timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_$o.log 2>&1
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['ms_per_step'],d['kernels']['mac_multi'])" gpurun_out/bench_$o.log
done
