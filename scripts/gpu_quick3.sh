#!/bin/bash
# parity + cfg4 and cfg5 bench lines (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 60 python scripts/one_step.py > ${P}_step.log 2>&1 || { echo "one_step failed rc=$?" >> ${P}_step.log; exit 1; }
timeout 300 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_bench.log 2>&1; echo "bench rc=$?" >> ${P}_bench.log
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_bench5.log 2>&1; echo "bench rc=$?" >> ${P}_bench5.log
