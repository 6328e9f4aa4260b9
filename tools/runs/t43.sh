#!/bin/bash
# final library (FOLD_INPLACE variant added, kernel unchanged): the whole GPU suite
OUT=gpurun_out/t43; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; echo "rc=$?" >> $OUT/ref.err
