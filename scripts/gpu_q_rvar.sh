#!/bin/bash
# quick2 + round variants (tag = $1, variants after)
cd $GRAFT_REPO_ROOT
T=$1
shift
bash scripts/gpu_quick2.sh $T
bash scripts/gpu_rvar.sh ${T}v "$@"
