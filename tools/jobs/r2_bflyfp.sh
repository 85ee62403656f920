# GPU job: FP64-quotient butterfly probe vs integer probe
set -x
python -c "
import sys; sys.path.insert(0,'.')
from paper_2310_16530_b200 import _native
for k in (1, 2, 3, 0): print(k, _native.ntt_butterfly_peak(k)/1e9)"
timeout 300 ncu --set full --clock-control none -k regex:"bfly_peak_fp" -s 13 -c 1 -o gpurun_out/bflyfp python -c "
import sys; sys.path.insert(0,'.')
from paper_2310_16530_b200 import _native
print(_native.ntt_butterfly_peak(2)/1e9, _native.ntt_butterfly_peak(3)/1e9)" > gpurun_out/ncu_bflyfp.log 2>&1; tail -2 gpurun_out/ncu_bflyfp.log
