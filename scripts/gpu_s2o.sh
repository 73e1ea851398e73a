#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 900 python -m pytest tests/test_gpu_sim.py tests/test_sim_pins.py -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 600 python scripts/sim_study.py --config 3 --depths 0,3 > ${P}_opp_cfg3.jsonl 2> ${P}_opp.err
timeout 600 python scripts/sim_study.py --config 3 --depths 0,3 --opportunistic >> ${P}_opp_cfg3.jsonl 2>> ${P}_opp.err
timeout 900 python scripts/sim_study.py --config 4 --jobs 3000 --depths 3 --opportunistic > ${P}_opp_cfg4.jsonl 2>> ${P}_opp.err
echo done > ${P}_done.txt
