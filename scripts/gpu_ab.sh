#!/bin/bash
# A/B of libcrius builds on one box (tag = $1, then variant names; "cur" = the in-tree build)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
shift
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = cur ]; then L=$PWD/paper_2403_16125_b200/libcrius.so; else L=$PWD/variants/$v; fi
  CRIUS_LIB=$L timeout 200 python scripts/round_bench.py --stats --configs ${CFGS:-4,5,3} >> ${P}_ab.log 2>&1
done
done
echo done > ${P}_done.txt
