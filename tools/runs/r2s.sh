#!/bin/bash
OUT=gpurun_out/${TAG:-r2s}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "query_split or degenerate or edge" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python tools/sanitize_case.py > $OUT/plain.log 2>&1 && \
  timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_case.py > $OUT/racecheck.log 2>&1
echo "racecheck_rc=$?" >> $OUT/racecheck.log
