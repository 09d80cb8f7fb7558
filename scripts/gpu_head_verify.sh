#!/bin/bash
# HEAD on a fresh box: full GPU suite, smoke(), the default bench line.
mkdir -p gpurun_out
T=gpurun_out/head
python -c "import __graft_entry__ as g; g.build()" > ${T}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > ${T}_pytest.log 2>&1; echo "rc=$?" >> ${T}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > ${T}_smoke.log 2>&1; echo "rc=$?" >> ${T}_smoke.log
timeout 1200 python bench.py > ${T}_bench.json 2> ${T}_bench.err; tail -c 1500 ${T}_bench.err > ${T}_bench.errtail; rm -f ${T}_bench.err
echo done > ${T}_done.txt
