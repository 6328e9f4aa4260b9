#!/bin/bash
OUT=gpurun_out/${TAG:-r2f}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "small_scan or invariances or scan_paths or stage_parity or cfg1 or code_operand" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/cfg4.json 2> $OUT/cfg4.err; echo "rc=$?" >> $OUT/cfg4.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/cfg3.json 2> $OUT/cfg3.err; echo "rc=$?" >> $OUT/cfg3.err

