#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round_paths.py tests/test_gpu_round_state.py tests/test_gpu_sim.py -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
bash scripts/gpu_ab.sh $1 v_prev cur
