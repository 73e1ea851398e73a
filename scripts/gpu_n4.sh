#!/bin/bash
# N-GPU check (tag = $1, N = $2): multi-GPU tests (NCCL + P2P exchange), bench lines NCCL vs P2P
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
N=$2
nvidia-smi topo -m > ${P}_topo.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu_nccl.py -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
for c in 4 5; do
  for g in nccl p2p; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 \
      bench.py --gpus $N --steps 20 --warmup 3 --config $c --gather $g > ${P}_n${N}_c${c}_${g}.json 2> ${P}_n${N}_c${c}_${g}.err
  done
done
echo done > ${P}_done.txt
