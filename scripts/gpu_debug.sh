#!/bin/bash
# full GPU suite against the -DCRIUS_DEBUG build (device-side bounds checks)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
export CRIUS_LIB=$PWD/variants/libcrius_debug.so
timeout 120 python scripts/sanitize_step.py > ${P}_dbgstep.log 2>&1 || { echo "failed rc=$?" >> ${P}_dbgstep.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > ${P}_dbgtests.log 2>&1; echo "rc=$?" >> ${P}_dbgtests.log
timeout 120 python scripts/one_step.py --config 4 >> ${P}_dbgstep.log 2>&1
timeout 300 python scripts/one_step.py --config 5 --reps 1 >> ${P}_dbgstep.log 2>&1
echo done >> ${P}_dbgstep.log
