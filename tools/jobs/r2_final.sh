# GPU job: default bench line (BASELINE metric) + config-2 primitive line + smoke
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_v9.log 2>&1; tail -c 400 gpurun_out/bench_v9.log
python bench.py --workload cfg2 > gpurun_out/bench_cfg2_v9.log 2>&1; tail -c 1500 gpurun_out/bench_cfg2_v9.log
