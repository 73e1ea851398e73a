#!/bin/bash
# round-end rehearsal (tag = $1): full GPU suite, smoke(), default bench line
cd $GRAFT_REPO_ROOT
P=gpurun_out/$1
timeout 1500 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc=$?" >> ${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "smoke rc=$?" >> ${P}_smoke.log
timeout 300 python bench.py > ${P}_bench.json 2> ${P}_bench.err; echo "bench rc=$?" >> ${P}_bench.err
timeout 300 python bench.py --impl reference > ${P}_ref.json 2> ${P}_ref.err
echo done > ${P}_done.txt
