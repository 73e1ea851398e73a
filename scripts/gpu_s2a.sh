#!/bin/bash
# session-2 check: full GPU suite (incl. 2-GPU NCCL + P2P exchange), estimate variants,
# N=2 bench lines NCCL vs fused P2P exchange (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
nvidia-smi topo -m > ${P}_topo.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
for v in v_minb3 v_w1 v_w1_minb3; do
  CRIUS_LIB=$PWD/variants/$v timeout 120 python scripts/est_bench.py --configs 4,5,4-pow2,3 >> ${P}_variants.log 2>&1
done
timeout 120 python scripts/est_bench.py --configs 4,5,4-pow2,3 >> ${P}_variants.log 2>&1
for c in 5 4; do
  for g in nccl p2p; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
      bench.py --gpus 2 --steps 20 --warmup 3 --config $c --gather $g > ${P}_n2_c${c}_${g}.json 2> ${P}_n2_c${c}_${g}.err
  done
done
echo done > ${P}_done.txt
