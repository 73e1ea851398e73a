#!/bin/bash
# fastest check: one_step (hang guard) + one bench line, no pytest (tag = $1, extra bench args after)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
shift
timeout 60 python scripts/one_step.py > ${P}_step.log 2>&1 || { echo "one_step failed rc=$?" >> ${P}_step.log; exit 1; }
timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > ${P}_bench.log 2>&1; echo "bench rc=$?" >> ${P}_bench.log
