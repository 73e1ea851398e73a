#!/bin/bash
# 2-GPU: NCCL parity test + bench at N=2 (torchrun) and N=1 for comparison
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
nvidia-smi topo -m > ${P}_topo.txt 2>&1
timeout 300 python -m pytest tests/test_multigpu_nccl.py -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 > ${P}_bench2.log 2>&1; echo "bench2 rc=$?" >> ${P}_bench2.log
timeout 300 python bench.py --steps 10 --warmup 3 --impl reference > ${P}_ref.log 2>&1; echo "ref rc=$?" >> ${P}_ref.log
