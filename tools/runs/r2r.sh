#!/bin/bash
OUT=gpurun_out/${TAG:-r2r}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --workload build --config 2 --steps 2 --warmup 1 > $OUT/build2.json 2> $OUT/build2.err; echo "rc=$?" >> $OUT/build2.err
timeout 900 python bench.py --workload build --config 4 --steps 1 --warmup 1 > $OUT/build4.json 2> $OUT/build4.err; echo "rc=$?" >> $OUT/build4.err
timeout 600 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
