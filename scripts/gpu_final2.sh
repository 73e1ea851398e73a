#!/bin/bash
# estimator A/B (v_prev vs in-tree) + round-end rehearsal (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
bash scripts/gpu_ab_est.sh $1 v_prev cur
bash scripts/gpu_final.sh $1
