#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 60 python scripts/one_step.py > ${P}_step.log 2>&1 || { echo "one_step failed" >> ${P}_step.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_assembly.py -x -q > ${P}_asm.log 2>&1; echo "asm rc=$?" >> ${P}_asm.log
timeout 300 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_assembly.py > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
