#!/bin/bash
# quick iteration: parity tests + one bench line (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 900 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > ${P}_bench.log 2>&1; echo "bench rc=$?" >> ${P}_bench.log
