#!/bin/bash
# round-kernel variants (tag = $1)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 200 python scripts/round_bench.py --stats >> ${P}_round.log 2>&1
for v in v_profseq v_seqw1 v_seqw2 v_seqw4; do
  CRIUS_LIB=$PWD/variants/$v timeout 200 python scripts/round_bench.py --stats >> ${P}_round.log 2>&1
done
timeout 200 python scripts/est_bench.py --configs 4,5,4-pow2,3 >> ${P}_est.log 2>&1
echo done > ${P}_done.txt
