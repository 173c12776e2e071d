for k in 2 3; do for r in 32 24 40 48; do
MPCORE_PANEL_ROWS=$r timeout 300 python bench.py --k $k --steps 6 --warmup 3 --no-cpu > gpurun_out/t.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/t.json')); print('k=$k rows=$r', '%.1f GF/s %.3f ms' % (d['value'], d['ms_per_step']))"
done; done
