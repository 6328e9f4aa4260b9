#!/bin/bash
OUT=gpurun_out/${TAG:-r2q}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "sharded or shards or query_split or nccl or degenerate or one_dimension or stage_parity" > $OUT/pytest_new.log 2>&1; echo "rc=$?" >> $OUT/pytest_new.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -s -p no:cacheprovider > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
