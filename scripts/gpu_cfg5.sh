#!/bin/bash
# cfg5 (96-layer GPT, S<=32, B sweep): bench + launch list
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 120 python scripts/one_step.py --config 5 > ${P}_step5.log 2>&1 || exit 1
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > ${P}_bench5.log 2>&1; echo "bench rc=$?" >> ${P}_bench5.log
timeout 300 python bench.py --config 4 --variant pow2 --steps 5 --warmup 3 --no-cpu-baseline > ${P}_bench4p.log 2>&1; echo "bench rc=$?" >> ${P}_bench4p.log
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > ${P}_bench3.log 2>&1; echo "bench rc=$?" >> ${P}_bench3.log
