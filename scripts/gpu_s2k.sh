#!/bin/bash
# NEXT-4 ablations: GPU parity + study (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 900 python -m pytest tests/test_gpu_round_state.py tests/test_gpu_sim.py tests/test_gpu_parity.py tests/test_gpu_round_paths.py tests/test_abi.py -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 600 python scripts/sim_study.py --config 3 --depths 3 --policies 0,1,2,3 > ${P}_ablation_cfg3.jsonl 2> ${P}_ablation.err
timeout 900 python scripts/sim_study.py --config 4 --jobs 3000 --depths 3 --policies 0,1,2,3 > ${P}_ablation_cfg4.jsonl 2>> ${P}_ablation.err
timeout 600 python scripts/sim_study.py --config 3 --depths 3 --policies 0 --deadlines 0.8 > ${P}_deadline_cfg3.jsonl 2>> ${P}_ablation.err
bash scripts/gpu_ab.sh $1 v_base cur
echo done > ${P}_done.txt
