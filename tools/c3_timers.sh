MPCORE_REFINE_TIMERS=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_2107_12550_b200.refine import refine_config3
for i in range(2):
    r = refine_config3()
    print(r['timings'], r['iterations'], file=sys.stderr)
"
