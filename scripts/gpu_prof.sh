#!/bin/bash
# ncu evidence for the bench command: launch list + full capture of the top kernels
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-flush"
timeout 200 $CMD > ${P}_plain.log 2>&1 || { echo "plain failed" >> ${P}_plain.log; exit 1; }
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${P}_launches.csv $CMD > ${P}_ncu1.log 2>&1
echo "ncu1 rc=$?" >> ${P}_plain.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_estimate|k_round_greedy" -s 2 -c 2 -o ${P}_full $CMD > ${P}_ncu2.log 2>&1
echo "ncu2 rc=$?" >> ${P}_plain.log
