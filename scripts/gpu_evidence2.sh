#!/bin/bash
# evidence (tag = $1): bench lines (+ unpipelined e2e), round stats, estimator alone, reference arm,
# launch list, full captures of k_estimate / k_round
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > ${P}_smi.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 > ${P}_bench4.json 2> ${P}_bench4.err
timeout 300 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline > ${P}_bench5.json 2> ${P}_bench5.err
timeout 300 python bench.py --config 4 --variant pow2 --steps 10 --warmup 3 --no-cpu-baseline > ${P}_bench4p.json 2> ${P}_bench4p.err
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > ${P}_bench3.json 2> ${P}_bench3.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > ${P}_ref4.json 2> ${P}_ref4.err
timeout 300 python bench.py --paper-stages --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_bench4ps.json 2> ${P}_bench4ps.err
timeout 300 python bench.py --config 5 --paper-stages --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_bench5ps.json 2> ${P}_bench5ps.err
timeout 300 python bench.py --assembly 1 --form 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > ${P}_benchasm.json 2> ${P}_benchasm.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-chunks 0 > ${P}_bench4_e2e0.json 2> ${P}_bench4_e2e0.err
timeout 300 python scripts/round_bench.py --configs 4,5,3 --stats > ${P}_round_stats.log 2>&1
timeout 300 python scripts/est_bench.py --configs 4,5,3,4-pow2 --reps 20 > ${P}_est.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-flush"
timeout 200 $CMD > ${P}_plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${P}_launches.csv $CMD > ${P}_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_estimate|7k_roundI" -s 2 -c 2 -o ${P}_full $CMD > ${P}_ncu2.log 2>&1
CMD5="python scripts/est_bench.py --configs 5 --reps 1"
timeout 200 $CMD5 > ${P}_plain5.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_estimate" -s 1 -c 1 -o ${P}_full5 $CMD5 > ${P}_ncu3.log 2>&1
echo done > ${P}_done.txt
