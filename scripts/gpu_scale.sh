#!/bin/bash
# strong scaling N = 1, 2, 4 on one box (tag = $1, configs in $2)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
NG=$(nvidia-smi -L | wc -l)
timeout 300 python -m pytest tests/test_multigpu_nccl.py -x -q > ${P}_nccl.log 2>&1; echo "rc=$?" >> ${P}_nccl.log
for cfg in $2; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > ${P}_c${cfg}_n1.json 2>&1
  for n in 2 4 8; do
    if [ $n -le $NG ]; then
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --config $cfg --gpus $n --steps 10 --warmup 3 > ${P}_c${cfg}_n$n.json 2>${P}_c${cfg}_n$n.err
    fi
  done
done
