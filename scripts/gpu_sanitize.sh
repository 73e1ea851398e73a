#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
TOOL=$2
timeout 120 python scripts/sanitize_step.py > ${P}_plain.log 2>&1 || exit 1
timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 9 python scripts/sanitize_step.py > ${P}_${TOOL}.log 2>&1
echo "rc=$?" >> ${P}_${TOOL}.log
