for c in 2147483647 1536 1024 700 0; do
MPCORE_NEXT_MAIN_COLS_DD=$c timeout 300 python bench.py --k 2 --steps 8 --warmup 3 --no-cpu > gpurun_out/t.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/t.json')); print('dd_cols=$c', '%.1f GF/s %.3f ms' % (d['value'], d['ms_per_step']))"
done
