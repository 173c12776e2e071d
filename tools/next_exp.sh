for k in 3 2 4; do for cfg in "X=1" "MPCORE_NEXT_ON_MAIN=1"; do
env $cfg timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/t.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/t.json')); print($k, '$cfg', '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), {a: round(b,2) for a,b in d['kernels_ms_per_step'].items()})"
done; done
