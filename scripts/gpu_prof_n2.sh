#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
CMD="python bench.py --config ${2:-5} --paper-stages --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-flush"
timeout 200 $CMD > ${P}_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_estimate" -s 1 -c 1 -o ${P}_n2 $CMD > ${P}_ncu.log 2>&1
echo "ncu rc=$?" >> ${P}_plain.log
