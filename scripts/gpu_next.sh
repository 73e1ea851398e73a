#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 300 python bench.py --assembly 1 --form 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_asm1.json 2>&1
timeout 300 python bench.py --assembly 1 --form 1 --tune --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_tune.json 2>&1
timeout 300 python bench.py --config 3 --assembly 1 --form 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_asm3.json 2>&1
