# exercise the N>1 code paths on one GPU (both ranks on device 0; replicas,
# not a measurement)
MPCORE_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu > gpurun_out/mr.json 2> gpurun_out/mr.err; echo rc=$?
tail -c 600 gpurun_out/mr.json; grep -i "error\|Traceback" gpurun_out/mr.err | head -5
MPCORE_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 2 --config 1 --steps 1 --warmup 1 --no-cpu > gpurun_out/mr1.json 2> gpurun_out/mr1.err; echo rc=$?
tail -c 300 gpurun_out/mr1.json
