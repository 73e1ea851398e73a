#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
CMD="python scripts/one_step.py --reps 2"
timeout 300 $CMD > ${P}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_round_greedy" -s 1 -c 1 -o ${P}_round $CMD > ${P}_ncu.log 2>&1
echo "rc=$?" >> ${P}_plain.log
