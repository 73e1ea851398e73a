#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
bash scripts/gpu_ab_est.sh $1 v_minb5 cur
