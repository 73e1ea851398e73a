#!/bin/bash
# source-level captures: k_round_greedy at cfg4, k_estimate at cfg5 (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
CMD="python scripts/one_step.py --reps 2"
timeout 300 $CMD > ${P}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_round_greedy" -s 1 -c 1 -o ${P}_round $CMD > ${P}_ncu.log 2>&1
CMD5="python scripts/est_bench.py --configs 5 --reps 1"
timeout 200 $CMD5 > ${P}_plain5.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_estimate" -s 1 -c 1 -o ${P}_est5 $CMD5 > ${P}_ncu5.log 2>&1
echo "rc=$?" >> ${P}_plain.log
