# GPU job: full gpu tests + default bench line (driver's command) + boot16
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_v11.log 2>&1; tail -c 600 gpurun_out/bench_v11.log
timeout 600 python tools/boot16.py > gpurun_out/boot16_v11.json 2>&1; tail -c 300 gpurun_out/boot16_v11.json
