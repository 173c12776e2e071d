# update-tile candidate masks vs whole-LU time (bench k, n = 2048)
run() { MPCORE_UPDATE_TILES=$2 timeout 300 python bench.py --k $1 --steps 5 --warmup 3 --no-cpu > gpurun_out/m.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/m.json')); print('k=$1 mask=$2', '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), 'upd %.3f step %.3f' % (d['roofline']['frac'], d['roofline']['whole_step_frac']))"; }
for m in 0x3e 0x08 0x20 0x28 0x40 0x48 0x68; do run 2 $m; done
for m in 0x08 0x40 0x48 0x02; do run 3 $m; done
