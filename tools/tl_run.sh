python tools/timeline.py 2 2048 400 > gpurun_out/tl_dd.txt 2>&1
python tools/timeline.py 3 2048 400 > gpurun_out/tl_td.txt 2>&1
MPCORE_NO_LOOKAHEAD=1 python tools/timeline.py 2 2048 400 > gpurun_out/tl_dd_nola.txt 2>&1
