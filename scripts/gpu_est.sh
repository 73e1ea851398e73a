#!/bin/bash
# estimate-kernel change: parity tests of the estimator, then estimate timings (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 60 python scripts/one_step.py > ${P}_step.log 2>&1 || { echo "one_step failed rc=$?" >> ${P}_step.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 120 python scripts/est_bench.py --configs 4,5,4-pow2 > ${P}_est.log 2>&1
