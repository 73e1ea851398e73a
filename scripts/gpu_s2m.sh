#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paper_stages.py tests/test_gpu_assembly.py -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
bash scripts/gpu_ab_est.sh $1 v_prev cur
