#!/bin/bash
# the scaling command at N = 1 (torchrun): config 4 through the native driver
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 1 --warmup 1 > /tmp/tr1.json 2>/tmp/tr1.err
echo "rc=$?"; tail -c 1500 /tmp/tr1.json; grep -v "NCCL INFO" /tmp/tr1.err | tail -3
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 1 --steps 1 --warmup 0 > /tmp/tr2.json 2>/tmp/tr2.err
echo "ref rc=$?"; tail -c 600 /tmp/tr2.json
