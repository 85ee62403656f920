# GPU job: re-check after container re-creation: gpu tests, smoke, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_recheck.log 2>&1; tail -c 600 gpurun_out/bench_recheck.log
