#!/bin/bash
OUT=gpurun_out/${TAG:-r2y}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/cfg4.json 2> $OUT/cfg4.err
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/cfg3.json 2> $OUT/cfg3.err
