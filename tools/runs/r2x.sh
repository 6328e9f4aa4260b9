#!/bin/bash
OUT=gpurun_out/${TAG:-r2x}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "small_scan or stage_parity or invariances or scan_paths or degenerate" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/cfg4.json 2> $OUT/cfg4.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall --variant 2 > $OUT/cfg4_v2.json 2> $OUT/cfg4_v2.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall --variant 8 > $OUT/cfg4_v8.json 2> $OUT/cfg4_v8.err
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/cfg3.json 2> $OUT/cfg3.err
timeout 900 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/cfg2.json 2> $OUT/cfg2.err
