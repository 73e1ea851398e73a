#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
CRIUS_LIB=$PWD/variants/trace.so timeout 120 python scripts/one_step.py --reps 1 > ${P}_trace.log 2>&1; echo "rc=$?" >> ${P}_trace.log
