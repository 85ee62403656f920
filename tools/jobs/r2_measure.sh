# GPU job: bench line with the integer roofline, butterfly peaks, ncu --set full of the top kernels
set -x
python bench.py > gpurun_out/bench2.log 2>&1; tail -c 600 gpurun_out/bench2.log
python -c "
import sys; sys.path.insert(0,'.')
from paper_2310_16530_b200 import _native
print('peak fast', _native.ntt_butterfly_peak(True)/1e9, 'full', _native.ntt_butterfly_peak(False)/1e9)
"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ntt2_fwd|k_ks_inner|k_mac_multi" -s 400 -c 8 -o gpurun_out/r20_full python tools/r20_once.py > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
