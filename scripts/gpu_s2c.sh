#!/bin/bash
# round-kernel change check (tag = $1): parity of the round paths + timing
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 200 python scripts/round_bench.py --stats >> ${P}_round.log 2>&1
CRIUS_LIB=$PWD/variants/v_profseq timeout 200 python scripts/round_bench.py --stats --configs 4 >> ${P}_round.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round_paths.py tests/test_gpu_round_state.py -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
echo done > ${P}_done.txt
