#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 900 python -m pytest tests/test_gpu_sim.py -x -q > ${P}_sim.log 2>&1; echo "rc=$?" >> ${P}_sim.log
