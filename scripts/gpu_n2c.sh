#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
bash scripts/gpu_tests1.sh $1 tests/test_gpu_paper_stages.py
for c in 4 5; do
  timeout 180 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --paper-stages --json-out ${P}_cfg${c}_paper.json > /dev/null 2>> ${P}_err.log
done
