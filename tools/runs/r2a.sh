#!/bin/bash
# round 2, first call: CFG4 bench line + ncu --set full of the CFG4 scan
OUT=gpurun_out/r2a; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/cfg4.json 2> $OUT/cfg4.err; echo "rc=$?" >> $OUT/cfg4.err
CMD="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-recall"
$CMD > $OUT/plain.log 2>&1 && \
 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"scan_imma" -s 4 -c 2 -o $OUT/full $CMD > $OUT/ncu_full.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_full.log
