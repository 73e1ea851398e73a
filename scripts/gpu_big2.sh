#!/bin/bash
# final-code multi-GPU lines (tag = $1): cfg5 x10 at N=1/4 (NCCL, P2P), cfg4/cfg5 at N=4 (NCCL, P2P)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517"
timeout 600 python bench.py --config 5 --scale 10 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_c5x10_n1.json 2> ${P}_c5x10_n1.err
timeout 600 $RUN bench.py --gpus 4 --config 5 --scale 10 --steps 5 --warmup 3 --no-e2e > ${P}_c5x10_n4_nccl.json 2> ${P}_c5x10_n4_nccl.err
timeout 600 $RUN bench.py --gpus 4 --config 5 --scale 10 --steps 5 --warmup 3 --no-e2e --gather p2p > ${P}_c5x10_n4_p2p.json 2> ${P}_c5x10_n4_p2p.err
for c in 4 5; do for g in nccl p2p; do
  timeout 300 $RUN bench.py --gpus 4 --steps 20 --warmup 3 --config $c --gather $g > ${P}_n4_c${c}_${g}.json 2> ${P}_n4_c${c}_${g}.err
done; done
echo done > ${P}_done.txt
