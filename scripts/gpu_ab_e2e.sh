#!/bin/bash
# A/B of the bench line incl. e2e (tag = $1, then variants; "cur" = in-tree build)
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
shift
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = cur ]; then L=$PWD/paper_2403_16125_b200/libcrius.so; else L=$PWD/variants/$v; fi
  echo "== $v" >> ${P}_abx.log
  CRIUS_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --config ${CFG:-4} >> ${P}_abx.log 2>> ${P}_abx.err
done
done
echo done > ${P}_done.txt
