#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_parity.py -k x10 -x -q > ${P}_x10test.log 2>&1; echo "rc=$?" >> ${P}_x10test.log
timeout 600 python bench.py --config 5 --scale 10 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_b5x10_n1.json 2>&1
if [ $NG -ge 4 ]; then
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29622 bench.py --config 5 --scale 10 --gpus 4 --steps 5 --warmup 3 > ${P}_b5x10_n4.json 2>${P}_b5x10_n4.err
fi
