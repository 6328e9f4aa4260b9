#!/bin/bash
# folded scan record widths: parity of the three plans, then CFG4 / CFG5-shard / CFG3 timing per plan
OUT=gpurun_out/t31; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "small_scan_identical or latency or fold" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 0 128 256; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall --variant $v > $OUT/cfg4_v$v.json 2> $OUT/cfg4_v$v.err
done
for v in 0 128 256; do
  timeout 600 python bench.py --config 5 --shard 0/8 --steps 5 --warmup 3 --no-cpu-baseline --no-recall --variant $v > $OUT/cfg5_v$v.json 2> $OUT/cfg5_v$v.err
done
