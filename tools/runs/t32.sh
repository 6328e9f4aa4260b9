#!/bin/bash
# folded scan epilogue reads only the valid columns: TMEM read peak (ubench), parity, CFG4 / CFG5-shard / CFG3 timing
OUT=gpurun_out/t32; mkdir -p $OUT
./tools/ubench/tmem_ld > $OUT/tmem_ld.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "small_scan_identical or latency or fold" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4.json 2> $OUT/cfg4.err
timeout 600 python bench.py --config 5 --shard 0/8 --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg5.json 2> $OUT/cfg5.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg3.json 2> $OUT/cfg3.err
