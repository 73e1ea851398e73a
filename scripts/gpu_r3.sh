#!/bin/bash
# round 1, call 3: parity tests, bench, ncu launch list + full capture of k_estimate / k_round_greedy
cd $GRAFT_REPO_ROOT
P=gpurun_out/r3
timeout 900 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > ${P}_bench.log 2>&1; echo "bench rc=$?" >> ${P}_bench.log
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-flush"
timeout 300 $CMD > ${P}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${P}_launches.csv $CMD > ${P}_ncu1.log 2>&1
echo "ncu1 rc=$?" >> ${P}_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_estimate|k_round_greedy" -c 2 -o ${P}_prof $CMD > ${P}_ncu2.log 2>&1
echo "ncu2 rc=$?" >> ${P}_plain.log
