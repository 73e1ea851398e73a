#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 900 python scripts/sim_study.py --config 3 --depths 0,1,3 > ${P}_study3.jsonl 2>&1
timeout 900 python scripts/sim_study.py --config 4 --jobs 3000 --depths 0,3 > ${P}_study4.jsonl 2>&1
