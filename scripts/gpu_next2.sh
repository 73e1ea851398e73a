#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 60 python scripts/one_step.py > ${P}_step.log 2>&1 || exit 1
for c in 4 5; do
  timeout 180 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --paper-stages --json-out ${P}_cfg${c}_paper.json > /dev/null 2>> ${P}_err.log
  timeout 180 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out ${P}_cfg${c}_uniform.json > /dev/null 2>> ${P}_err.log
done
