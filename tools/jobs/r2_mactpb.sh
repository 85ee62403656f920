# GPU job: plane MAC with 128 threads x 2 coefficients per thread vs 256 x 1 (bit-exactness + ResNet20)
set -x
HCNN_OPTIONS=mac_tpb=128 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
HCNN_OPTIONS=mac_tpb=128,tma_stages=3 timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_layers.py tests/test_gpu_hashes.py -m gpu -x -q 2>&1 | tail -2
for o in mac_tpb=256 mac_tpb=128 mac_tpb=128,tma_stages=3; do
  HCNN_OPTIONS=$o timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_$o.log 2>&1
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],d['ms_per_step'],d['kernels']['mac_multi'])" gpurun_out/bench_$o.log
done
