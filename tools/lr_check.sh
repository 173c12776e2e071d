timeout 900 python -m pytest tests/test_gpu_long_residual.py tests/test_gpu_config3.py tests/test_gpu_ffi.py -x -q 2>&1 | tail -3
bash tools/c3_timers.sh 2>&1 | tail -14
timeout 600 python bench.py --config 3 --steps 5 --warmup 2 > gpurun_out/c3.json 2> gpurun_out/c3.err; tail -2 gpurun_out/c3.err
python -c "
import json; d=json.load(open('gpurun_out/c3.json')); print(d['value'], d['timings_s'], d['result']['iterations'], d['result']['stop_reason'])"
