bash tools/lr_check.sh
mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:long_residual_warp -c 1 -o gpurun_out/prof/long_residual python -c "
import sys; sys.path.insert(0,'.')
from paper_2107_12550_b200.refine import refine_config3
refine_config3()
" > gpurun_out/prof/lr.log 2>&1; tail -3 gpurun_out/prof/lr.log
