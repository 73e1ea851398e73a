#!/bin/bash
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
shift
for v in "$@"; do
  CRIUS_LIB=$PWD/variants/$v timeout 120 python scripts/est_bench.py --configs 4,5,4-pow2 >> ${P}_variants.log 2>&1
done
timeout 120 python scripts/est_bench.py --configs 4,5,4-pow2 >> ${P}_variants.log 2>&1
