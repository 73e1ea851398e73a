#!/bin/bash
# round-kernel variants: one bench line each (CRIUS_LIB override), tag = $1, variants after
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
shift
timeout 60 python scripts/one_step.py > ${P}_step.log 2>&1 || { echo "one_step failed rc=$?" >> ${P}_step.log; exit 1; }
for v in "$@"; do
  echo "== $v" >> ${P}_rvar.log
  CRIUS_LIB=$PWD/variants/$v timeout 60 python scripts/one_step.py >> ${P}_rvar.log 2>&1 || echo "variant $v failed" >> ${P}_rvar.log
  CRIUS_LIB=$PWD/variants/$v timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out ${P}_$v.json > /dev/null 2>> ${P}_rvar.log
done
