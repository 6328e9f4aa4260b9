#!/bin/bash
# ncu --set full of the small-K scan at CFG4 (main scan launch)
OUT=gpurun_out/${TAG:-r2c}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CMD="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-recall"
$CMD > $OUT/plain.log 2>&1 && \
 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"scan_small" -s 5 -c 2 -o $OUT/full $CMD > $OUT/ncu_full.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_full.log
