#!/bin/bash
# full GPU tests + bench at N=1 and N=2 (tag = $1); needs gpurun --gpus 2
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 60 python scripts/one_step.py > ${P}_step.log 2>&1 || { echo "one_step failed rc=$?" >> ${P}_step.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 240 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > ${P}_n1.log 2>&1; echo "rc=$?" >> ${P}_n1.log
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > ${P}_n2.log 2>&1; echo "rc=$?" >> ${P}_n2.log
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --config 5 --gpus 2 --steps 10 --warmup 3 > ${P}_n2c5.log 2>&1; echo "rc=$?" >> ${P}_n2c5.log
