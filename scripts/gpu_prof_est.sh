#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
CFG=${2:-4}
CMD="python scripts/est_bench.py --configs $CFG --reps 2"
timeout 120 $CMD > ${P}_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_estimate" -s 2 -c 1 -o ${P}_est $CMD > ${P}_ncu.log 2>&1
echo "ncu rc=$?" >> ${P}_plain.log
