#!/bin/bash
# folded scan: flagged pairs deferred to a tail phase (per-CTA record region)
OUT=gpurun_out/t42; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "small_scan_identical or latency" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4_S.json 2> $OUT/cfg4_S.err
timeout 600 python bench.py --config 5 --shard 0/8 --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg5_S.json 2> $OUT/cfg5_S.err
