#!/bin/bash
# bench at N=1 and N=2 (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
python -c "import paper_2403_16125_b200 as p; print(p.lib())" > ${P}_load.log 2>&1
timeout 240 python bench.py --steps 10 --warmup 3 > ${P}_n1.log 2>&1; echo "rc=$?" >> ${P}_n1.log
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > ${P}_n2.log 2>&1; echo "rc=$?" >> ${P}_n2.log
