#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 60 python scripts/one_step.py > ${P}_step.log 2>&1 || { echo "one_step failed" >> ${P}_step.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_round_state.py -x -q > ${P}_state.log 2>&1; echo "rc=$?" >> ${P}_state.log
timeout 600 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_bench.log 2>&1
