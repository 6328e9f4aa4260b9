#!/bin/bash
OUT=gpurun_out/${TAG:-r2p}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/cfg4.json 2> $OUT/cfg4.err; echo "rc=$?" >> $OUT/cfg4.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/cfg3.json 2> $OUT/cfg3.err; echo "rc=$?" >> $OUT/cfg3.err
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/cfg2.json 2> $OUT/cfg2.err; echo "rc=$?" >> $OUT/cfg2.err
